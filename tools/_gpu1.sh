timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "small_blocks or fixture or streamed or solve_shift or contour_pass" > gpurun_out/t_small.log 2>&1; echo small=$?; tail -3 gpurun_out/t_small.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['phase_ms_per_step'], round(d['e2e']['value'],1))"
FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace.log 2>&1; grep -v "contour pass\|rayleigh" gpurun_out/trace.log | tail -16
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
