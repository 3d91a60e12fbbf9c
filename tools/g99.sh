O=gpurun_out/g99; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c1" > $O/pytest_c1.txt 2>&1 || exit 0
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
FKV_TC_PINGPONG=1 timeout 600 python -m pytest tests/test_gpu_parity2.py -q -k "pingpong" > $O/pytest_pp.txt 2>&1
for i in 1 2; do for v in base wa; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
