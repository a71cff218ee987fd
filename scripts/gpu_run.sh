mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/slab.jsonl
for ny in 4096 2048 1024 512; do
  for op in poisson mom_v; do timeout 300 python scripts/kbench.py --solve $op --nx 4096 --ny $ny >> gpurun_out/slab.jsonl 2>> gpurun_out/slab.err; echo $ny$op=$? >> $S; done
done
