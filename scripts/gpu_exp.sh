#!/bin/sh
# variant experiment: parity of libch_b200_$V.so first, then isolated 4096^2 solves
# against the default library (two repetitions).  V=<variant> sh scripts/gpu_exp.sh
mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
L=$PWD/paper_1811_11842_b200/libch_b200_$V.so
CHB_LIB=$L timeout 400 python -m pytest tests/test_gpu_parity.py -q -x \
  -k "forced_strips or (one_step_matches_oracle) or virtual_slabs_match or three_steps" > gpurun_out/t_$V.log 2>&1; echo t_$V=$? >> $S
if grep -q " passed" gpurun_out/t_$V.log && ! grep -q "failed\|error" gpurun_out/t_$V.log; then
  for rep in 1 2; do
    for lib in default $V; do
      LL=$L; [ $lib = default ] && LL=$PWD/paper_1811_11842_b200/libch_b200.so
      for op in mom_v poisson; do
        CHB_LIB=$LL timeout 180 python scripts/kbench.py --solve $op --stride 1 | sed "s/^{/{\"variant\": \"$lib\", /" >> gpurun_out/kb_$V.jsonl 2>&1
      done
    done
  done
fi
echo done >> $S
