# Round bench suite (1 GPU): bench lines for every config, both tcgen05 kernels on C2, the reference arm, a 2-rank
set -x
O=${1:-gpurun_out/r02}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q --timeout 600 > $O/pytest_gpu.txt 2>&1
timeout 600 python bench.py --steps 10 > $O/bench_c2_none.json 2> $O/err_c2_none.txt
FKV_KERNEL=3 timeout 400 python bench.py --steps 10 --no-cpu-baseline --no-deferred > $O/bench_c2_none_rows.json 2> $O/err_c2_rows.txt
timeout 400 python bench.py --mode deferred --steps 5 --no-cpu-baseline > $O/bench_c2_deferred.json 2> $O/err_c2_def.txt
timeout 300 python bench.py --config c1 --steps 10 --no-cpu-baseline > $O/bench_c1_none.json 2> $O/err_c1.txt
timeout 500 python bench.py --config c3 --steps 3 --no-e2e --no-cpu-baseline > $O/bench_c3_none.json 2> $O/err_c3.txt
timeout 400 python bench.py --config c5 --steps 5 --no-cpu-baseline > $O/bench_c5_none.json 2> $O/err_c5.txt
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4_none.json 2> $O/err_c4.txt
timeout 400 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_c2_reference.json 2> $O/err_ref.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --no-cpu-baseline --no-deferred --no-e2e > $O/bench_c2_2ranks_1gpu.json 2> $O/err_2ranks.txt
FKV_NVTX=1 timeout 400 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_none.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-deferred --no-graph > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ra_tc_kernel -s 3 -c 1 -o $O/prof_c2_none python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-deferred --no-graph > /dev/null 2>&1
FKV_KERNEL=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:ra_rows -s 3 -c 1 -o $O/prof_c2_rows python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-deferred --no-graph > /dev/null 2>&1
