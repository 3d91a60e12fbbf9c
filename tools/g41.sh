O=gpurun_out/g41; mkdir -p $O
FKV_KERNEL=3 timeout 600 python bench.py --config c3 --steps 3 --no-e2e --no-cpu-baseline > $O/c3_rows.json 2> $O/c3_rows.err
FKV_KERNEL=3 timeout 300 python tools/timeline_rows.py --help > $O/tlr_help.txt 2>&1
