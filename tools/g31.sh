mkdir -p gpurun_out/g31
for fl in 0 1; do FKV_ROWS_FLAGS=$fl FKV_PIECE_FRAC=0.5 timeout 120 python tools/timeline_rows.py --tiles 14 > gpurun_out/g31/tl_$fl.txt 2>&1; done
FKV_ROWS_FLAGS=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "c1_parity or page_sizes or c2_full" > gpurun_out/g31/pytest_fl1.txt 2>&1
