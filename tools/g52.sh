O=gpurun_out/g52; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench.json 2>$O/bench.err
FKV_NVTX=1 timeout 400 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_none.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-deferred --no-graph > /dev/null 2>&1
