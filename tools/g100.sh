O=gpurun_out/sweep_s3; mkdir -p $O
for r in 16 8; do
  for n in 4 16 64 256; do
    timeout 900 python bench.py --config sweep --rank $r --fanout $n --steps 3 --warmup 3 --no-e2e --no-cpu-baseline \
      --no-deferred --no-graph > $O/sweep_r${r}_n${n}.json 2> $O/sweep_r${r}_n${n}.err
  done
done
