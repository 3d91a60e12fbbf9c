O=gpurun_out/g55; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -k "test_c1_parity and (tc-none or tc128-none)" > $O/sanitizer_racecheck.txt 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity2.py -q -k "needle" > $O/sanitizer_racecheck_needle.txt 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench.json 2>$O/bench.err
