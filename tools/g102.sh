O=gpurun_out/g102; mkdir -p $O
for i in 1 2; do for v in s0 s20 s50 s100 s200; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
