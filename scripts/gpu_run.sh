# one gpurun call: tests, persistent vs per-launch solves, bench
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 600 python -m pytest tests -m gpu -q -k "persistent" > gpurun_out/pytest_persist.log 2>&1; echo pytest_persist=$? >> $S
for ps in 0 1; do for op in poisson mom_v; do CHB_PERSIST=$ps timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"persist\": $ps, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done; done
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
CHB_PERSIST=1 timeout 900 python bench.py > gpurun_out/bench_persist.log 2>&1; echo bench_persist=$? >> $S
