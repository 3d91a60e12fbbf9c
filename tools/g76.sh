O=gpurun_out/g76; mkdir -p $O
timeout 300 python tools/step_skip.py > $O/skip.txt 2>&1
