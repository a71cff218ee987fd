#!/bin/sh
# One gpurun call: smoke, the full GPU test suite, the headline bench and the
# configs[1] / configs[2] bench lines.  Outputs in gpurun_out/.
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
if [ "${SKIP_BENCH:-0}" = 0 ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> $S
fi
for c in 1 2; do
  timeout 600 python bench.py --config $c --matvec 0 > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err
  echo bench_c$c=$? >> $S
done
