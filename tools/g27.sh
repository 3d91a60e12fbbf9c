mkdir -p gpurun_out/g27
timeout 120 tools/ub_mix > gpurun_out/g27/ub_mix.txt 2>&1
