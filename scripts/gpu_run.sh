# one gpurun call: tests, solve timing, bench, ncu of the dominant sweep + px, launch list
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl gpurun_out/*.ncu-rep
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for op in poisson mom_v; do timeout 300 python scripts/kbench.py --solve $op >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
V="python scripts/kbench.py --solve mom_v"
timeout 300 $V > gpurun_out/plain_v.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 3000 -c 2 -o gpurun_out/prof_cgs_v -f $V > gpurun_out/ncu_full_v.log 2>&1; echo ncufv=$? >> $S
timeout 900 ncu --set full --clock-control none -k regex:k_cgs_px -s 50 -c 1 -o gpurun_out/prof_px -f $V > gpurun_out/ncu_px.log 2>&1; echo ncupx=$? >> $S
P="python scripts/kbench.py --solve poisson"
timeout 300 $P > gpurun_out/plain_p.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 3000 -c 2 -o gpurun_out/prof_cgs_p -f $P > gpurun_out/ncu_full_p.log 2>&1; echo ncufp=$? >> $S
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_b.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_bench_head.csv $B > gpurun_out/ncu_lb.log 2>&1; echo ncul=$? >> $S
du -sh gpurun_out >> $S
