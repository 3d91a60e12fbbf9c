O=gpurun_out/g106; mkdir -p $O
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_tl.so timeout 200 python tools/timeline.py --mode deferred --page 128 --tiles 6 --detail 20 --first 18 > $O/tl_def.txt 2>&1
