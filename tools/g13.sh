mkdir -p gpurun_out/g13
for i in 1 2 3; do FKV_HANG_DIAG=1 timeout 150 python tools/repro_bench.py 32 8 nosync > gpurun_out/g13/nosync_$i.txt 2>&1; done
timeout 120 python tools/timeline_rows.py --tiles 24 > gpurun_out/g13/tl.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/g13/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/g13/bench.json 2> gpurun_out/g13/bench.err
