timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_eig.csv python tools/eig_timing.py 192 > /dev/null 2>&1; echo rc=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:"chol_sm" -c 1 -o gpurun_out/chol_sm python tools/eig_timing.py 192 > /dev/null 2>&1; echo rc=$?
