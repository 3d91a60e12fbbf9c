O=gpurun_out/g60; mkdir -p $O
for v in s32 s47 base s16; do
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python tools/timeline.py --mode none --page 128 --tiles 2 --detail 20 > $O/tl_$v.txt 2>&1
done
