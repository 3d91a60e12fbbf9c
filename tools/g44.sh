O=gpurun_out/g44; mkdir -p $O
for pf in 0 2 4 8; do
  FKV_TC_L2PF=$pf timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_pf$pf.json 2>$O/err_$pf.txt
done
FKV_TC_L2PF=4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "c2_full or c1" > $O/pytest.txt 2>&1
