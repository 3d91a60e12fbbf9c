set -x
mkdir -p gpurun_out/g2
timeout 120 tools/ub_mix > gpurun_out/g2/ub_mix.txt 2>&1
timeout 120 python -X faulthandler -c "
import faulthandler, sys; faulthandler.dump_traceback_later(90, exit=True)
sys.argv=['bench.py','--steps','2','--warmup','3','--no-cpu-baseline','--no-e2e']
import runpy; runpy.run_path('bench.py', run_name='__main__')
" > gpurun_out/g2/bench_rows.json 2> gpurun_out/g2/bench_rows.err
timeout 120 python bench.py --config c1 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/g2/bench_c1_rows.json 2> gpurun_out/g2/bench_c1_rows.err
