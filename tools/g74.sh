O=gpurun_out/g74; mkdir -p $O
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 --block 100 --detail 30 > $O/tl_b100_d30.txt 2>&1
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 50 --block 100 --first 28 > $O/tl_b100_t.txt 2>&1
