O=gpurun_out/g79; mkdir -p $O
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_carve$i.json 2>$O/err_c$i.txt
FKV_NO_CARVEOUT=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_nocarve$i.json 2>$O/err_n$i.txt
done
