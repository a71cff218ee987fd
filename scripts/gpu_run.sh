# asynchronous p/x: parity + timing
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests -m gpu -q -k "async_px or deferred or persistent" > gpurun_out/pytest_apx.log 2>&1; echo pytest_apx=$? >> $S
for ap in 0 1; do for op in poisson mom_v; do CHB_PXASYNC=$ap timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"apx\": $ap, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done; done
CHB_PXASYNC=1 timeout 900 python bench.py > gpurun_out/bench_apx.log 2>&1; echo bench_apx=$? >> $S
