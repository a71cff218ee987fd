# per-rank slab shapes of the strong-scaling runs (4096 x 4096/N), isolated solves
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
for ny in 4096 2048 1024 512; do for op in poisson mom_v; do timeout 300 python scripts/kbench.py --nx 4096 --ny $ny --solve $op >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done; done
echo done >> $S
