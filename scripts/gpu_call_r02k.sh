#!/bin/sh
# re-entry verification of HEAD: smoke, GPU suite, headline bench
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> $S
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
