#!/bin/sh
# P2P combine tests (cooperative emulation, virtual slabs, loopback ranks),
# early-start sweep A/B (CHB_EARLY) on isolated solves and the headline bench.
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_xrank.py tests/test_multirank_loopback.py tests/test_gpu_parity.py -q -x --durations=5 > gpurun_out/t_p2p.log 2>&1; echo t_p2p=$? >> $S
CHB_EARLY=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/t_early.log 2>&1; echo t_early=$? >> $S
for e in 0 1 0 1; do for op in mom_v poisson; do
  CHB_EARLY=$e timeout 300 python scripts/kbench.py --solve $op --stride 1 >> gpurun_out/kb_early$e.jsonl 2>&1
done; done
CHB_EARLY=1 timeout 900 python bench.py --no-cpu > gpurun_out/bench_early1.json 2> gpurun_out/bench_early1.err; echo bench1=$? >> $S
timeout 900 python bench.py --no-cpu > gpurun_out/bench_early0.json 2> gpurun_out/bench_early0.err; echo bench0=$? >> $S
