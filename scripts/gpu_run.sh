mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
for k in 0 256 4352 12544; do
  for op in poisson mom_v; do CHB_SKEW=$k timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"skew\": $k, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo $k$op=$? >> $S; done
done
