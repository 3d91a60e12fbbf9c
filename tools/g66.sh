O=gpurun_out/g66; mkdir -p $O
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred > $O/bench_e2e.json 2>$O/err_e2e.txt
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_base$i.json 2>$O/err_base$i.txt
FKV_DIAG_NOSTAGE=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_nostage$i.json 2>$O/err_nostage$i.txt
done
