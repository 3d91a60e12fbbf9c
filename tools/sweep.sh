# configs[4] rank x fan-out sweep (1 GPU): one bench line per point into $O
O=${1:-gpurun_out/sweep}; mkdir -p $O
for r in 16 8 64; do
  for n in 4 16 64 256; do
    timeout 900 python bench.py --config sweep --rank $r --fanout $n --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
      --no-deferred --no-graph > $O/sweep_r${r}_n${n}.json 2> $O/sweep_r${r}_n${n}.err
  done
done
