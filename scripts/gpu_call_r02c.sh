#!/bin/sh
# Round 2 (session 2): R25 momentum guess -- smoke, parity suite, 4096^2
# per-step diagnostics and the headline bench.
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x --durations=10 > gpurun_out/gpu_parity.log 2>&1; echo parity=$? >> $S
timeout 900 python scripts/diag_steps.py --n 4096 --steps 25 > gpurun_out/diag_4096.jsonl 2>&1; echo diag=$? >> $S
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> $S
