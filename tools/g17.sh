mkdir -p gpurun_out/g17
timeout 120 tools/ub_tile > gpurun_out/g17/ub_tile.txt 2>&1
