#!/bin/sh
# joint u/v momentum sweep: parity tests, then the headline bench with and without it
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "joint or one_step or forced_strips_all or three_steps" > gpurun_out/t_uv.log 2>&1; echo tests=$? >> $S
timeout 900 python bench.py --no-cpu --matvec 0 > gpurun_out/bench_uv1.json 2> gpurun_out/bench_uv1.err; echo bench1=$? >> $S
CHB_UV=0 timeout 900 python bench.py --no-cpu --no-e2e --matvec 0 > gpurun_out/bench_uv0.json 2> gpurun_out/bench_uv0.err; echo bench0=$? >> $S
