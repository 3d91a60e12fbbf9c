mkdir -p gpurun_out/g28
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "c1_parity or page_sizes or random_suite or c2_full" > gpurun_out/g28/pytest_quick.txt 2>&1
FKV_PIECE_FRAC=0.5 timeout 120 python tools/timeline_rows.py --tiles 16 > gpurun_out/g28/tl_05.txt 2>&1
FKV_PIECE_FRAC=0.15 timeout 120 python tools/timeline_rows.py --tiles 16 > gpurun_out/g28/tl_015.txt 2>&1
FKV_PIECE_FRAC=0.3 timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g28/tl_03.txt 2>&1
