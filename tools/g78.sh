O=gpurun_out/g78; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity2.py -q -x -k "split_phases or host_entry or decode_loop" > $O/pytest.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench$i.json 2>$O/err$i.txt
done
