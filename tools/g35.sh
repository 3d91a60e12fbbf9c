mkdir -p gpurun_out/g35
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity2.py -x -q --timeout 200 > gpurun_out/g35/pytest.txt 2>&1
for f in 0.5 0.3 0.2; do FKV_PIECE_FRAC=$f timeout 120 python tools/timeline_rows.py --tiles 16 > gpurun_out/g35/tl_$f.txt 2>&1; done
