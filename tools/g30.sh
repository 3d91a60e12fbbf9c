mkdir -p gpurun_out/g30
for fl in 0 24; do FKV_ROWS_FLAGS=$fl FKV_PIECE_FRAC=0.5 timeout 120 python tools/timeline_rows.py --tiles 14 > gpurun_out/g30/tl_$fl.txt 2>&1; done
