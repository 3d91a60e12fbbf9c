O=gpurun_out/g77; mkdir -p $O
timeout 200 python tools/timeline.py --mode deferred --page 128 --tiles 12 --detail 20 --first 16 > $O/tl_def.txt 2>&1
