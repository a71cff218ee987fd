mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 900 python -m pytest tests -m gpu -q -s -k "refinement or smooth_rhs" > gpurun_out/pytest_ref.log 2>&1; echo ref=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
