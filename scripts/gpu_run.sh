# one gpurun call: wave-count experiment, tests
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl gpurun_out/*.ncu-rep
for w in 1 2 3 4; do for op in poisson mom_v; do CHB_WAVES=$w timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"waves\": $w, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done; done
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
