timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "gevp or tridiag or feast_solve or shrinking" > gpurun_out/t14.log 2>&1; echo t14=$?; tail -1 gpurun_out/t14.log; grep -E "^E |FAILED" gpurun_out/t14.log | head -5
for v in 11 12 21 22 41 14; do
  FEAST_EIGVALS=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tri_eig" -c 12 --csv --log-file gpurun_out/ev_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "EIGVALS=$v"; python tools/launches.py gpurun_out/ev_$v.csv | head -3
done
for w in 2 4; do
  FEAST_EIGVECS_WPB=$w timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tri_eigvecs" -c 6 --csv --log-file gpurun_out/evv_$w.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "EIGVECS_WPB=$w"; python tools/launches.py gpurun_out/evv_$w.csv | head -2
done
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench14.log 2>&1; tail -1 gpurun_out/bench14.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['phase_ms_per_step'], round(d['e2e']['value'],1))"
