mkdir -p gpurun_out/g20
timeout 400 /usr/local/cuda/bin/cuda-gdb -batch -ex "set cuda break_on_launch none" -ex run -ex "info cuda kernels" -ex "bt" -ex "x/6i \$pc-32" -ex "info line *\$pc" --args python tools/timeline_rows.py --tiles 4 > gpurun_out/g20/gdb.txt 2>&1
