mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 900 python -m pytest tests/test_multirank_loopback.py -x -q > gpurun_out/loopback.log 2>&1; echo loopback=$? >> $S
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
