python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1; echo plain=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"bt_sweep_bulk" -s 3 -c 1 -o gpurun_out/r01_sweep_bulk_cfg2_full python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1; echo full=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_bench_launches_cfg2_v2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo list=$?
