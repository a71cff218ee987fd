#!/bin/sh
# CH apply variants (CTAs per SM x ring depth): parity of each library, then the
# isolated applies at 4096^2 / 16384^2, two rounds.  VARIANTS="a b" sh scripts/gpu_exp_ch.sh
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
P=$PWD/paper_1811_11842_b200
for v in $VARIANTS; do
  CHB_LIB=$P/libch_b200_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x \
    -k "forced_strips or one_step_matches_oracle or apply" > gpurun_out/t_$v.log 2>&1; echo t_$v=$? >> $S
done
for rep in 1 2; do
  for v in default $VARIANTS; do
    L=$P/libch_b200_$v.so; [ $v = default ] && L=$P/libch_b200.so
    CHB_LIB=$L timeout 200 python scripts/matvec_sweep.py --sizes 4096 16384 | grep '"ch"' | sed "s/^{/{\"variant\": \"$v\", /" >> gpurun_out/mv_ch.jsonl
  done
done
echo done >> $S
