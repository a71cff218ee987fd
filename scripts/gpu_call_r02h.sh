#!/bin/sh
# bench contract test + the profile pass (headline bench, launch list, ncu).
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bench_contract.py -q > gpurun_out/t_bench.log 2>&1; echo t_bench=$? > gpurun_out/tests_status.txt
sh scripts/gpu_profile.sh
