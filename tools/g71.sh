O=gpurun_out/g71; mkdir -p $O
for i in 1 2; do for v in base early; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
FKV_DIAG_NOSTAGE=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_nostage.json 2>$O/err_nostage.txt
