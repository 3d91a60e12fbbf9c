O=gpurun_out/g84; mkdir -p $O
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE OK')" > $O/smoke.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 300 python bench.py > $O/bench_default.json 2> $O/bench_default.err
