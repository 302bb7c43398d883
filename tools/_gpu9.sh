timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/t9.log 2>&1; echo t9=$?; tail -1 gpurun_out/t9.log; grep -E "^E |FAILED" gpurun_out/t9.log | head -5
FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace.log 2>&1; grep -v "contour pass\|rayleigh" gpurun_out/trace.log | tail -14
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['phase_ms_per_step'], d['e2e'])"
