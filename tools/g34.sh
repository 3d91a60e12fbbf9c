mkdir -p gpurun_out/g34
for f in 0.5 0.3 0.2; do FKV_PIECE_FRAC=$f timeout 120 python tools/timeline_rows.py --tiles 4 > gpurun_out/g34/tl_$f.txt 2>&1; done
