O=gpurun_out/g82; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity2.py -q -k "pingpong" > $O/pytest_pp.txt 2>&1
