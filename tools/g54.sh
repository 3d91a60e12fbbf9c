O=gpurun_out/g54; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
timeout 300 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_merge.txt 2>&1
FKV_NO_MERGE=1 timeout 300 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_nomerge.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred > $O/bench_merge.json 2>$O/bench_merge.err
FKV_NO_MERGE=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_nomerge.json 2>$O/bench_nomerge.err
timeout 300 python bench.py --config c5 --steps 5 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_c5.json 2>$O/bench_c5.err
