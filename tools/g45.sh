O=gpurun_out/g45; mkdir -p $O
FKV_TC_ROWS=128 timeout 600 python bench.py --config c3 --steps 3 --no-e2e --no-cpu-baseline > $O/c3_r128.json 2> $O/c3_r128.err
FKV_TC_ROWS=128 timeout 300 python bench.py --steps 10 --no-e2e --no-cpu-baseline --no-deferred > $O/c2_r128.json 2> $O/c2_r128.err
timeout 600 python bench.py --config c3 --steps 3 --no-e2e --no-cpu-baseline > $O/c3_r64.json 2> $O/c3_r64.err
