O=gpurun_out/g63; mkdir -p $O
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 70 --detail 0 > $O/tl_d0.txt 2>&1
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 --detail 28 > $O/tl_d28.txt 2>&1
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 --detail 58 > $O/tl_d58.txt 2>&1
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 70 --block 100 --detail 0 > $O/tl_b100.txt 2>&1
