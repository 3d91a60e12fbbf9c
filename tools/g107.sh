O=gpurun_out/g107; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c1 and deferred" > $O/pytest_c1.txt 2>&1 || exit 0
timeout 900 python -m pytest tests -m gpu -q -k "deferred" > $O/pytest_def.txt 2>&1
for i in 1 2; do for v in norb rb; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 400 python bench.py --mode deferred --steps 5 --no-cpu-baseline --no-e2e > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
