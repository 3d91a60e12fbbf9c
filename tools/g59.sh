O=gpurun_out/g59; mkdir -p $O
for v in base vB vD vE vF; do
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python tools/timeline.py --mode none --page 128 --tiles 2 --detail 20 > $O/tl_$v.txt 2>&1
done
for v in vB vD vE vF; do
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c2_full or c1" > $O/pytest_$v.txt 2>&1
done
