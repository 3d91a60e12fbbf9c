O=gpurun_out/g83; mkdir -p $O
timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e > $O/c2.json 2>$O/c2.err
timeout 600 python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/c4.json 2> $O/c4.err
