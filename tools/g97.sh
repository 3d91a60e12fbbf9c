O=gpurun_out/g97; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > $O/smoke.txt 2>&1
for i in 1 2; do
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench$i.json 2>$O/err$i.txt
done
bash tools/variants.sh tl "-DFKV_TIMELINE=1" > $O/variants.txt 2>&1
FKV_LIB_PATH=paper_2604_06370_b200/variants/libforkkv_tl.so timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl.txt 2>&1
timeout 120 python tools/timeline.py --mode none --page 128 --tiles 2 > $O/tl_prod.txt 2>&1
