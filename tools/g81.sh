O=gpurun_out/g81; mkdir -p $O
FKV_TC_PINGPONG=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c1" > $O/pytest_pp_c1.txt 2>&1
FKV_TC_PINGPONG=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity2.py -q > $O/pytest_pp.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_base$i.json 2>$O/err_b$i.txt
FKV_TC_PINGPONG=1 timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_pp$i.json 2>$O/err_p$i.txt
done
FKV_TC_PINGPONG=1 timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 --detail 20 > $O/tl_pp.txt 2>&1
