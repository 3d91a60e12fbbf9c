O=gpurun_out/g98; mkdir -p $O
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_sm.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1 or c2_full" > $O/pytest.txt 2>&1
for i in 1 2; do for v in base sm; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
