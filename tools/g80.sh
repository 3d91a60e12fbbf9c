O=gpurun_out/g80; mkdir -p $O
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl.txt 2>&1
