# one gpurun call: tests, L2-prefetch distance sweep, matvec sweeps, bench
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl gpurun_out/matvec.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for pf in 0 8 16 32; do for op in poisson mom_u; do CHB_PF=$pf timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"pf\": $pf, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done; done
timeout 600 python scripts/matvec_sweep.py > gpurun_out/matvec.jsonl 2> gpurun_out/matvec.err; echo matvec=$? >> $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
