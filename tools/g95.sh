O=gpurun_out/g95; mkdir -p $O
FKV_TC_PINGPONG=1 timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu_pp.txt 2>&1
