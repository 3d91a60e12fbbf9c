O=gpurun_out/g73; mkdir -p $O
for b in 0 40 100 140; do
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 --block $b > $O/tl_b$b.txt 2>&1
done
