# one gpurun call: tests, kernel timing (solves + steps), bench, ncu of the CG kernels
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for op in poisson mom_u; do timeout 300 python scripts/kbench.py --solve $op >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kbs$op=$? >> $S; done
timeout 300 python scripts/kbench.py --config 3 >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kb=$? >> $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
P="python scripts/kbench.py --solve poisson"
timeout 300 $P > gpurun_out/plain_p.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs -s 6000 -c 17 -o gpurun_out/prof_cgs_p -f $P > gpurun_out/ncu_full_p.log 2>&1; echo ncufp=$? >> $S
V="python scripts/kbench.py --solve mom_v"
timeout 300 $V > gpurun_out/plain_v.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 3000 -c 2 -o gpurun_out/prof_cgs_v -f $V > gpurun_out/ncu_full_v.log 2>&1; echo ncufv=$? >> $S
