# warp-decoupled sweep: parity + timing
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl gpurun_out/*.ncu-rep
timeout 900 python -m pytest tests -m gpu -q -k "sweep_sync_variants" > gpurun_out/pytest_ws.log 2>&1; echo pytest_ws=$? >> $S
for ws in 0 1; do for op in poisson mom_v; do CHB_WS=$ws timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"ws\": $ws, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done; done
CHB_WS=1 timeout 900 python bench.py > gpurun_out/bench_ws.log 2>&1; echo bench_ws=$? >> $S
