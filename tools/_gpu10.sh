timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "hermitian" > gpurun_out/t10.log 2>&1; echo t10=$?; tail -2 gpurun_out/t10.log; grep -E "^E |FAILED" gpurun_out/t10.log | head -6
