nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t11.log 2>&1; echo t11=$?; tail -1 gpurun_out/t11.log; grep -E "^E |FAILED" gpurun_out/t11.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d.get('phase_ms_per_step'), d['e2e'], d['roofline'], d['cpu_baseline'], d['clocks'])"
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_ref.log
