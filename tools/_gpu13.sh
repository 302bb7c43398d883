timeout 300 python -m pytest tests/test_gpu_csr_ingest.py -x -q > gpurun_out/t13a.log 2>&1; echo t13a=$?; tail -3 gpurun_out/t13a.log; grep -E "^E |FAILED|Error" gpurun_out/t13a.log | head -12
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t13.log 2>&1; echo t13=$?; tail -1 gpurun_out/t13.log; grep -E "^E |FAILED" gpurun_out/t13.log | head -5
FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace13.log 2>&1; grep -v "contour pass\|rayleigh" gpurun_out/trace13.log | tail -14
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench13.log 2>&1; tail -1 gpurun_out/bench13.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['phase_ms_per_step'], d['e2e'])"
