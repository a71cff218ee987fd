#!/bin/sh
# pipelined polls: parity + full-size + loopback tests, then the headline bench
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_multirank_loopback.py tests/test_bench_contract.py -q -x > gpurun_out/t_poll.log 2>&1; echo tests=$? >> $S
for op in mom_v poisson; do timeout 300 python scripts/kbench.py --solve $op --stride 1 >> gpurun_out/kb_poll.jsonl 2>&1; done
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> $S
