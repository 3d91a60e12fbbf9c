O=gpurun_out/g42; mkdir -p $O
export FKV_KERNEL=3 FKV_DIAG_SKIP_SMALL=1
for f in 0 64 128 192 216; do
  FKV_ROWS_FLAGS=$f timeout 300 python tools/timeline_rows.py --tiles 12 > $O/tl_$f.txt 2>&1
done
