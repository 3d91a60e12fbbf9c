O=gpurun_out/g56; mkdir -p $O
timeout 300 python tools/timeline.py --mode none --page 128 --tiles 70 --detail 30 > $O/tl.txt 2>&1
timeout 300 python tools/timeline.py --mode none --page 128 --tiles 4 --block 77 > $O/tl77.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ra_tc_kernel -s 3 -c 1 -o $O/prof python tools/timeline.py --mode none --page 128 --tiles 2 > $O/ncu.log 2>&1
ncu -i $O/prof.ncu-rep --page raw --csv > $O/raw.csv 2>&1
ncu -i $O/prof.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>&1
timeout 300 python bench.py --steps 10 --no-cpu-baseline > $O/bench.json 2>$O/bench.err
