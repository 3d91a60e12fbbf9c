O=gpurun_out/g48; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_rank.py -q > $O/pytest_rank.txt 2>&1
bash tools/sweep.sh $O
