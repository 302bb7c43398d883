timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "random_block or fixture or warm or determinism" > gpurun_out/t3.log 2>&1; echo t3=$?; tail -2 gpurun_out/t3.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['phase_ms_per_step'], d['e2e'])"
FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace.log 2>&1; grep -v "contour pass\|rayleigh" gpurun_out/trace.log | tail -12
