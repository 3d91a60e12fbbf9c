mkdir -p gpurun_out/g7
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ra_rows -s 3 -c 1 -o gpurun_out/g7/prof_rows python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-deferred --no-graph > gpurun_out/g7/ncu.log 2>&1
timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/g7/bench.json 2> gpurun_out/g7/bench.err
