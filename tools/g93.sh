O=gpurun_out/g93; mkdir -p $O
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_base$i.json 2>$O/err_b$i.txt
FKV_DIAG_NOSTAGE=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_nostage$i.json 2>$O/err_n$i.txt
done
