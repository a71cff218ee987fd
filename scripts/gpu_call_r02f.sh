#!/bin/sh
# BASELINE configs[4]: 16384^2 for its configured 10 steps on one B200
# (per-step time, Krylov iterations, field ranges).
mkdir -p gpurun_out
timeout 6000 python scripts/diag_steps.py --n 16384 --steps 10 > gpurun_out/diag_16384_10.jsonl 2>&1; echo diag=$? > gpurun_out/status.txt
