#!/bin/sh
# Final verification: smoke (2 steps), the whole GPU suite, configs[1] and
# configs[2] bench lines with the final build.
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
for c in 1 2; do
  timeout 600 python bench.py --config $c --matvec 0 > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err; echo bench_c$c=$? >> $S
done
