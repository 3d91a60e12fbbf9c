O=gpurun_out/g92; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity2.py -q -k "newest_rows" > $O/pytest.txt 2>&1
