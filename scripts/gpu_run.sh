# one gpurun call: tests, solve timing, bench, ncu of the pressure sweep
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for op in poisson mom_u; do timeout 300 python scripts/kbench.py --solve $op >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
P="python scripts/kbench.py --solve poisson"
timeout 300 $P > gpurun_out/plain_p.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 6000 -c 2 -o gpurun_out/prof_cgs_p -f $P > gpurun_out/ncu_full_p.log 2>&1; echo ncufp=$? >> $S
