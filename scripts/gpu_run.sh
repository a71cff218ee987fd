# one gpurun call: tests, solve timing variants, bench
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for r3 in 0 1; do for op in poisson mom_u; do CHB_ROWS3=$r3 timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"rows3\": $r3, /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done; done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_solve_p.csv python scripts/kbench.py --solve poisson > gpurun_out/ncu_l.log 2>&1; echo ncul=$? >> $S
