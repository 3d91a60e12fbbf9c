mkdir -p gpurun_out/g5
timeout 120 python tools/repro_bench.py 32 6 nosync > gpurun_out/g5/nosync.txt 2>&1
for pf in 0 2 4 8; do FKV_ROWS_PREFETCH=$pf timeout 120 python tools/timeline_rows.py --tiles 24 > gpurun_out/g5/tl_pf$pf.txt 2>&1; done
timeout 200 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/g5/bench.json 2> gpurun_out/g5/bench.err
