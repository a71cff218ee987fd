mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 900 python -m pytest tests -m gpu -x -q -k "persistent" > gpurun_out/gpu_tests_persist.log 2>&1; echo ptests=$? >> $S
rm -f gpurun_out/kbench.jsonl
for p in 0 1; do
  for op in poisson mom_v; do CHB_PERSIST=$p timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"persist\": $p, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo $p$op=$? >> $S; done
done
for p in 0 1; do CHB_PERSIST=$p timeout 300 python scripts/kbench.py --solve poisson --config 2 | sed "s/^{/{\"persist\": $p, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done
