#!/bin/sh
# cost of the true-residual refinement passes (R21) at 4096^2: the same 6 steps with refine = 0 / 1 / 2
mkdir -p gpurun_out
for r in 0 1 2; do
  timeout 300 python scripts/diag_steps.py --n 4096 --steps 6 --refine $r | sed "s/^{/{\"refine\": $r, /" >> gpurun_out/refine_cost.jsonl
done
