mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 900 python -m pytest tests/test_multirank_loopback.py -x -q > gpurun_out/loopback.log 2>&1; echo loopback=$? >> $S
