mkdir -p gpurun_out/g33
FKV_DIAG_SKIP_SMALL=1 FKV_PIECE_FRAC=0.5 timeout 120 python tools/timeline_rows.py --tiles 40 > gpurun_out/g33/tl.txt 2>&1
