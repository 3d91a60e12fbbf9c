O=gpurun_out/g64; mkdir -p $O
timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/c3_k2.json 2> $O/c3_k2.err
FKV_KERNEL=3 timeout 600 python bench.py --config c3 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/c3_k3.json 2> $O/c3_k3.err
FKV_KERNEL=3 timeout 600 python bench.py --config c5 --steps 5 --no-e2e --no-cpu-baseline > $O/c5_k3.json 2> $O/c5_k3.err
FKV_KERNEL=3 timeout 600 python bench.py --config c4 --steps 3 --no-e2e --no-cpu-baseline > $O/c4_k3.json 2> $O/c4_k3.err
