O=gpurun_out/g88; mkdir -p $O
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_base$i.json 2>$O/err_b$i.txt
FKV_STAGE_CARVEOUT=100 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_cv$i.json 2>$O/err_c$i.txt
done
