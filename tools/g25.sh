mkdir -p gpurun_out/g25
FKV_PIECE_FRAC=0.15 timeout 120 python tools/timeline_rows.py --tiles 20 > gpurun_out/g25/tl.txt 2>&1
