# one gpurun call: tests, matvec sweeps, kernel timing, bench, ncu of the CH apply
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl gpurun_out/matvec.jsonl
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> $S
timeout 1500 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
timeout 600 python scripts/matvec_sweep.py > gpurun_out/matvec.jsonl 2> gpurun_out/matvec.err; echo matvec=$? >> $S
CHB_CH_TILE=1 timeout 600 python scripts/matvec_sweep.py --sizes 4096 > gpurun_out/matvec_tile.jsonl 2>> gpurun_out/matvec.err; echo matvec_tile=$? >> $S
timeout 300 python scripts/kbench.py --config 3 >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kb=$? >> $S
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$? >> $S
M="python scripts/matvec_sweep.py --sizes 4096 --reps 5"
timeout 300 $M > gpurun_out/plain_m.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ch_rm -c 2 -o gpurun_out/prof_ch -f $M > gpurun_out/ncu_ch.log 2>&1; echo ncuch=$? >> $S
