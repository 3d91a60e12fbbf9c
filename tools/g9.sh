mkdir -p gpurun_out/g9
timeout 60 tools/ub_fill2 > gpurun_out/g9/ub_fill2.txt 2>&1
for i in 1 2 3 4; do FKV_HANG_DIAG=1 timeout 150 python tools/repro_bench.py 32 8 nosync > gpurun_out/g9/nosync_$i.txt 2>&1; done
