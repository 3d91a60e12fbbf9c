mkdir -p gpurun_out/g21
timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g21/tl.txt 2>&1
FKV_PIECE_FRAC=0.3 timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g21/tl_f03.txt 2>&1
FKV_PIECE_FRAC=1.0 timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g21/tl_f10.txt 2>&1
