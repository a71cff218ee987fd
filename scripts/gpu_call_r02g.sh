#!/bin/sh
# Sweep tail: per-CTA trace by dispatch order on the SM, then claimed tiles
# with skewed strip heights (CHB_SKEWA) A/B on isolated solves + parity.
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
T=$PWD/paper_1811_11842_b200/libch_b200_trace.so
for op in mom_v poisson; do nb=592; [ $op = poisson ] && nb=888
  CHB_LIB=$T timeout 300 python scripts/trace_sweep.py --solve $op --nb $nb >> gpurun_out/trace_order.jsonl 2>&1
  CHB_LIB=$T CHB_SKEWA=0.06 timeout 300 python scripts/trace_sweep.py --solve $op --nb $nb >> gpurun_out/trace_order_skew.jsonl 2>&1
done; echo trace=$? >> $S
for a in 0 0.03 0.06 0.1 -0.05 0 0.06; do for op in mom_v poisson; do
  echo "{\"skew\": \"$a\"}" >> gpurun_out/kb_skew.jsonl
  CHB_SKEWA=$a timeout 300 python scripts/kbench.py --solve $op --stride 1 >> gpurun_out/kb_skew.jsonl 2>&1
done; done; echo kb=$? >> $S
CHB_SKEWA=0.06 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "not 25_steps and not 50_steps" > gpurun_out/t_skew.log 2>&1; echo t_skew=$? >> $S
# CH apply with 4 CTAs/SM (<= 128 registers) vs the default 3
for v in "" _ch4; do
  CHB_LIB=$PWD/paper_1811_11842_b200/libch_b200$v.so timeout 300 python scripts/matvec_sweep.py --sizes 4096 16384 > gpurun_out/mv$v.jsonl 2>&1
done; echo mv=$? >> $S
