O=gpurun_out/g65; mkdir -p $O
for ov in 22 32 44 60; do
  FKV_ITEM_OVERHEAD=$ov timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_ov$ov.txt 2>&1
done
for pt in 24 28 36; do
  FKV_PIECE_TILES=$pt timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_pt$pt.txt 2>&1
done
