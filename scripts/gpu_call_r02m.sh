#!/bin/sh
# CTA width experiment (CHB_NTHR 64 / 96 vs 128): parity first, then isolated 4096^2 solves
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
for v in n64 n96; do
  CHB_LIB=$PWD/paper_1811_11842_b200/libch_b200_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "forced_strips_all or (one_step_matches_oracle and 130)" > gpurun_out/t_$v.log 2>&1; echo t_$v=$? >> $S
done
for rep in 1 2; do
for v in default n64 n96; do
  L=$PWD/paper_1811_11842_b200/libch_b200_$v.so; [ $v = default ] && L=$PWD/paper_1811_11842_b200/libch_b200.so
  if [ $v = default ] || grep -q "passed" gpurun_out/t_$v.log; then
    for op in mom_v poisson; do
      CHB_LIB=$L timeout 300 python scripts/kbench.py --solve $op --stride 1 | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/kb_width.jsonl 2>&1
    done
  fi
done
done
echo done >> $S
