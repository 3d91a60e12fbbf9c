# Round bench suite (1 GPU): bench lines for every config, ncu launch list and full profiles of the main kernel.
set -x
mkdir -p gpurun_out/r
timeout 400 python bench.py --steps 10 > gpurun_out/r/bench_c2_none.json 2> gpurun_out/r/err_c2_none.txt
timeout 400 python bench.py --mode deferred --steps 5 > gpurun_out/r/bench_c2_deferred.json 2> gpurun_out/r/err_c2_def.txt
timeout 300 python bench.py --config c1 --steps 10 > gpurun_out/r/bench_c1_none.json 2> gpurun_out/r/err_c1.txt
timeout 400 python bench.py --config c3 --steps 3 --no-e2e > gpurun_out/r/bench_c3_none.json 2> gpurun_out/r/err_c3.txt
timeout 400 python bench.py --config c5 --steps 5 > gpurun_out/r/bench_c5_none.json 2> gpurun_out/r/err_c5.txt
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-e2e > gpurun_out/r/bench_c4_none.json 2> gpurun_out/r/err_c4.txt
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r/bench_c2_reference.json 2> gpurun_out/r/err_ref.txt
timeout 400 ncu --set full --import-source on --clock-control none -k regex:ra_tc_kernel -s 3 -c 1 -o gpurun_out/r/prof_c2_none python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 400 ncu --set full --import-source on --clock-control none -k regex:ra_tc_kernel -s 3 -c 1 -o gpurun_out/r/prof_c2_deferred python bench.py --mode deferred --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"ra_|combine" -s 96 -c 96 --csv --log-file gpurun_out/r/launches_c2_none.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
