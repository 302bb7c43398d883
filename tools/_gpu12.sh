FEAST_TRACE=2 timeout 300 python tools/e2e_trace.py cfg2 > gpurun_out/trace.log 2>&1; grep -v "contour pass\|rayleigh" gpurun_out/trace.log | tail -40
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_bench_launches_cfg2_v4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1; echo list=$?
python tools/launches.py gpurun_out/r01_bench_launches_cfg2_v4.csv > gpurun_out/r01_bench_launches_cfg2_v4_summary.txt 2>&1; head -40 gpurun_out/r01_bench_launches_cfg2_v4_summary.txt
