timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gevp or fixture or residual or determinism or warm or truncation" > gpurun_out/t7.log 2>&1; echo t7=$?; tail -1 gpurun_out/t7.log; grep -E "^E |FAILED" gpurun_out/t7.log | head -5
timeout 120 python tools/eig_timing.py 64 160 192 > gpurun_out/eig.log 2>&1; cat gpurun_out/eig.log
FEAST_TRI=k timeout 120 python tools/eig_timing.py 192 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['phase_ms_per_step'], round(d['e2e']['value'],1))"
