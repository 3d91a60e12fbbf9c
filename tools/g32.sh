mkdir -p gpurun_out/g32
FKV_PIECE_FRAC=0.5 timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g32/tl_all.txt 2>&1
FKV_DIAG_SKIP_SMALL=1 FKV_PIECE_FRAC=0.5 timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g32/tl_noprivate.txt 2>&1
FKV_DIAG_SKIP_SMALL=1 FKV_PIECE_FRAC=0.2 timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g32/tl_noprivate02.txt 2>&1
