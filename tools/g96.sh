O=gpurun_out/g96; mkdir -p $O
git_rev=none
for i in 1 2; do for v in base notl; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e --no-deferred > $O/bench_${v}$i.json 2>$O/err_${v}$i.txt
done; done
for v in base notl; do
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_$v.so timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_$v.txt 2>&1
done
