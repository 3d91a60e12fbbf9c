O=gpurun_out/g105; mkdir -p $O
for i in 1 2; do for v in base vspin; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
