for v in 224 228 218 128 118; do
  FEAST_EIGVALS=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tri_eigvals" -c 6 --csv --log-file gpurun_out/ev_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "EIGVALS=$v"; python tools/launches.py gpurun_out/ev_$v.csv | head -1
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t15.log 2>&1; echo t15=$?; tail -1 gpurun_out/t15.log; grep -E "^E |FAILED" gpurun_out/t15.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke15.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench15.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench15.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['phase_ms_per_step'], round(d['e2e']['value'],1), d['gpu_launches'], d['clocks'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_bench_launches_cfg2_v5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu5.log 2>&1; echo list=$?
python tools/launches.py gpurun_out/r01_bench_launches_cfg2_v5.csv > gpurun_out/r01_bench_launches_cfg2_v5_summary.txt 2>&1; head -30 gpurun_out/r01_bench_launches_cfg2_v5_summary.txt
FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace15.log 2>&1; grep -A12 "warm ---" gpurun_out/trace15.log | grep -v "contour pass\|rayleigh"
