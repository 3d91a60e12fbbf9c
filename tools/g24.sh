mkdir -p gpurun_out/g24
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "c1_parity or page_sizes or random_suite or c2_full" > gpurun_out/g24/pytest_quick.txt 2>&1
for f in 0.15 0.08 0.3; do FKV_PIECE_FRAC=$f timeout 120 python tools/timeline_rows.py --tiles 8 > gpurun_out/g24/tl_$f.txt 2>&1; done
