timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "small_blocks or fixture or streamed or solve_shift or contour_pass" > gpurun_out/t_small.log 2>&1; echo small=$?; tail -2 gpurun_out/t_small.log
FEAST_TRACE=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_e2e.csv python tools/e2e_trace.py cfg2 > /dev/null 2>&1; echo rc=$?
FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace.log 2>&1; grep -v "contour pass\|rayleigh" gpurun_out/trace.log | tail -12
