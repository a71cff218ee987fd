mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
rm -f gpurun_out/kbench.jsonl
for sp in 1 2 3 4; do
  for op in poisson mom_v; do CHB_SPLIT=$sp timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"split\": $sp, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo $sp$op=$? >> $S; done
done
