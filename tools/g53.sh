O=gpurun_out/g53; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
for v in nolazy lazy; do
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_$v.txt 2>&1
  FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_$v.json 2>$O/bench_$v.err
done
