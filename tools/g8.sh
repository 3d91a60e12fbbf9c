mkdir -p gpurun_out/g8
for i in 1 2 3; do FKV_HANG_DIAG=1 timeout 150 python tools/repro_bench.py 32 8 nosync > gpurun_out/g8/nosync_$i.txt 2>&1; done
timeout 120 tools/ub_fill > gpurun_out/g8/ub_fill.txt 2>&1
