mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 900 python -m pytest tests/test_bench_contract.py -x -q > gpurun_out/contract.log 2>&1; echo contract=$? >> $S
