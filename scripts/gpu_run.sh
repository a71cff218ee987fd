# one gpurun call: tests, kernel-variant timing, bench, ncu of the fused CG sweep
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for v in 3 2; do CHB_VEC=$v timeout 300 python scripts/kbench.py --config 3 >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kb$v=$? >> $S; done
CHB_PDL=0 timeout 300 python scripts/kbench.py --config 3 >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kbnopdl=$? >> $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
P="python scripts/prof_step.py --config 3 --steps 1"
timeout 300 $P > gpurun_out/plain_p.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 3000 -c 2 -o gpurun_out/prof_cgs -f $P > gpurun_out/ncu_full.log 2>&1; echo ncuf=$? >> $S
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 36000 -c 2 -o gpurun_out/prof_cgs_p -f $P > gpurun_out/ncu_full_p.log 2>&1; echo ncufp=$? >> $S
