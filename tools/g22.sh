mkdir -p gpurun_out/g22
FKV_HANG_DIAG=1 timeout 150 python tools/repro_bench.py 32 4 nosync > gpurun_out/g22/nosync.txt 2>&1
timeout 120 python tools/timeline_rows.py --tiles 16 > gpurun_out/g22/tl.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity2.py -x -q --timeout 600 > gpurun_out/g22/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred > gpurun_out/g22/bench.json 2> gpurun_out/g22/bench.err
