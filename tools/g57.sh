O=gpurun_out/g57; mkdir -p $O
for v in base s1 s2 s4 s8 s12 s15 s16 s31; do
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_$v.txt 2>&1
done
FKV_TC_ROWS=128 timeout 300 python tools/timeline.py --mode none --page 128 --tiles 40 --detail 20 > $O/tl_r128.txt 2>&1
for v in base s3 s12 s15 s16; do
  FKV_TC_ROWS=128 FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_r128_$v.txt 2>&1
done
