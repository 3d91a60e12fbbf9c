O=gpurun_out/g70; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.txt 2>&1
timeout 300 python tools/host_overhead.py > $O/host.txt 2>&1
for i in 1 2 3; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench$i.json 2>$O/err$i.txt
done
