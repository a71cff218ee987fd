#!/bin/sh
# One gpurun call: smoke, the full GPU test suite, a memcheck pass over small
# parity cases (new kernels), and the headline bench.  Outputs in gpurun_out/.
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "(test_one_step_matches_oracle and 64-64) or test_operator_applies or test_moving_fluid or (test_virtual_slabs_match_single_slab and 2-1-1)" \
  > gpurun_out/memcheck.log 2>&1; echo memcheck=$? >> $S
if [ "${SKIP_BENCH:-0}" = 0 ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> $S
fi
for c in 1 2; do
  timeout 600 python bench.py --config $c --matvec 0 > gpurun_out/bench_config$c.json 2> gpurun_out/bench_config$c.err
  echo bench_c$c=$? >> $S
done
