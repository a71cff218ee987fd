mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for op in poisson mom_v mom_u; do timeout 300 python scripts/kbench.py --solve $op >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
