mkdir -p gpurun_out/g16
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ra_rows -s 3 -c 1 -o gpurun_out/g16/prof_rows python tools/timeline_rows.py --tiles 4 > gpurun_out/g16/ncu.log 2>&1
ncu -i gpurun_out/g16/prof_rows.ncu-rep --page raw --csv > gpurun_out/g16/raw.csv 2>&1
ncu -i gpurun_out/g16/prof_rows.ncu-rep --page details --csv > gpurun_out/g16/details.csv 2>&1
