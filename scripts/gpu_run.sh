mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
rm -f gpurun_out/kbench.jsonl
for d in 64 32; do
  for op in poisson mom_v; do CHB_DEFER=$d timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"m\": $d, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo $d$op=$? >> $S; done
done
