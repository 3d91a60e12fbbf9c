O=gpurun_out/g36; mkdir -p $O
timeout 300 python tools/step_breakdown.py > $O/breakdown.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred > $O/bench.json 2> $O/bench.err
