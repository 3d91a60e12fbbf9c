O=gpurun_out/g49; mkdir -p $O
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred > $O/bench.json 2>$O/bench.err
FKV_BENCH_EVENTS_IN_TIMED=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_ev.json 2>$O/bench_ev.err
