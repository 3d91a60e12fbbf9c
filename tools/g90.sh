O=gpurun_out/g90; mkdir -p $O
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_klf16.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity2.py -q -k "deferred" > $O/pytest_klf16.txt 2>&1
for i in 1 2; do for v in base klf16; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 400 python bench.py --mode deferred --steps 5 --no-cpu-baseline --no-e2e > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_klf16.so timeout 200 python tools/timeline.py --mode deferred --page 128 --tiles 2 --detail 20 --first 16 > $O/tl_klf16.txt 2>&1
