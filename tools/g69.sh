O=gpurun_out/g69; mkdir -p $O
nproc > $O/nproc.txt; cat /proc/cpuinfo | grep 'model name' | head -1 >> $O/nproc.txt
timeout 300 python tools/host_overhead.py > $O/host.txt 2>&1
for i in 1 2 3; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-deferred --no-e2e > $O/bench$i.json 2>$O/err$i.txt
done
