O=gpurun_out/g89; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity2.py tests/test_seq_split.py -q > $O/pytest.txt 2>&1
for i in 1 2 3; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench$i.json 2>$O/err$i.txt
done
