timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t17.log 2>&1; echo t17=$?; tail -1 gpurun_out/t17.log; grep -E "^E |FAILED" gpurun_out/t17.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke17.log 2>&1; echo smoke=$?
timeout 400 python bench.py > gpurun_out/bench17.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench17.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_bench_launches_cfg2_v6.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu6.log 2>&1; echo list=$?
python tools/launches.py gpurun_out/r01_bench_launches_cfg2_v6.csv > gpurun_out/r01_bench_launches_cfg2_v6_summary.txt 2>&1; head -16 gpurun_out/r01_bench_launches_cfg2_v6_summary.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"tri_eigvals" -s 3 -c 1 -o gpurun_out/r01_tri_eigvals_222_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_ev.log 2>&1; echo evfull=$?
FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace17.log 2>&1; grep -A14 "warm ---" gpurun_out/trace17.log | grep -v "contour pass\|rayleigh"
