O=gpurun_out/g61; mkdir -p $O
for v in s32 s32vB s32vG; do
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 120 python tools/timeline.py --mode none --page 128 --tiles 40 --detail 20 > $O/tl_$v.txt 2>&1
done
FKV_L2_EVICT=0 FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_s32.so timeout 120 python tools/timeline.py --mode none --page 128 --tiles 40 --detail 20 > $O/tl_s32_noevict.txt 2>&1
