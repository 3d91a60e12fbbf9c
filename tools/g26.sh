mkdir -p gpurun_out/g26
FKV_PIECE_FRAC=0.5 timeout 120 python tools/timeline_rows.py --tiles 20 > gpurun_out/g26/tl.txt 2>&1
