set -x
mkdir -p gpurun_out/g1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/g1/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/g1/bench_rows.json 2> gpurun_out/g1/bench_rows.err
FKV_KERNEL=2 timeout 300 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/g1/bench_tc.json 2> gpurun_out/g1/bench_tc.err
timeout 300 python tools/timeline_rows.py --tiles 40 > gpurun_out/g1/timeline_rows.txt 2>&1
