O=gpurun_out/g62; mkdir -p $O
for v in s12 s28 s44 s3 s35; do
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 --detail 20 > $O/tl_$v.txt 2>&1
done
