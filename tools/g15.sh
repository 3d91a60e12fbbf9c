mkdir -p gpurun_out/g15
for pf in 0 2 3 5; do FKV_ROWS_PREFETCH=$pf timeout 120 python tools/timeline_rows.py --tiles 12 > gpurun_out/g15/tl_pf$pf.txt 2>&1; done
FKV_HANG_DIAG=1 timeout 150 python tools/repro_bench.py 32 6 nosync > gpurun_out/g15/nosync.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity2.py tests/test_gpu_project.py -x -q --timeout 600 > gpurun_out/g15/pytest_gpu.txt 2>&1
