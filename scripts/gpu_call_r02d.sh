#!/bin/sh
# Full GPU suite (goldens regenerated for R25), then the profile pass
# (headline bench, launch lists, ncu --set full of the top kernels).
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$? > gpurun_out/tests_status.txt
sh scripts/gpu_profile.sh
