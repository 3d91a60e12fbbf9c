mkdir -p gpurun_out/g18
FKV_HANG_DIAG=1 timeout 150 python tools/repro_bench.py 32 6 nosync > gpurun_out/g18/nosync.txt 2>&1
for pf in 0 3; do FKV_ROWS_PREFETCH=$pf timeout 120 python tools/timeline_rows.py --tiles 16 > gpurun_out/g18/tl_pf$pf.txt 2>&1; done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/g18/pytest_gpu.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred > gpurun_out/g18/bench.json 2> gpurun_out/g18/bench.err
