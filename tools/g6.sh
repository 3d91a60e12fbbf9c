mkdir -p gpurun_out/g6
timeout 60 tools/ub_bulk4 > gpurun_out/g6/ub_bulk4.txt 2>&1
timeout 120 python tools/timeline_rows.py --tiles 24 > gpurun_out/g6/tl_cpasync.txt 2>&1
FKV_ROWS_FLAGS=1 timeout 120 python tools/timeline_rows.py --tiles 24 > gpurun_out/g6/tl_bulk.txt 2>&1
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/g6/pytest_gpu.txt 2>&1
