O=gpurun_out/g103; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench$i.json 2>$O/err$i.txt
done
