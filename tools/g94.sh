O=gpurun_out/g94; mkdir -p $O
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 4 --detail 0 > $O/tl_d0.txt 2>&1
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 4 --detail 0 --block 60 > $O/tl_d0_b60.txt 2>&1
