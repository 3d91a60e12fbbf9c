mkdir -p gpurun_out/g19
FKV_HANG_DIAG=1 timeout 150 python tools/repro_bench.py 32 4 nosync > gpurun_out/g19/nosync.txt 2>&1
for pf in 0 3; do FKV_ROWS_PREFETCH=$pf timeout 120 python tools/timeline_rows.py --tiles 16 > gpurun_out/g19/tl_pf$pf.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity2.py -x -q --timeout 600 > gpurun_out/g19/pytest_gpu.txt 2>&1
