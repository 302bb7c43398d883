for v in 224 222 212 312 412 422 122 314; do
  FEAST_EIGVALS=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tri_eigvals" -c 6 --csv --log-file gpurun_out/ev_$v.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
  echo "EIGVALS=$v $(python tools/launches.py gpurun_out/ev_$v.csv | head -1)"
done
