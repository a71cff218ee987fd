# one gpurun call: tests, kernel-variant timing, launch list, ncu of the momentum CG kernels
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> $S
for v in 2 1 0; do CHB_VEC=$v timeout 300 python scripts/kbench.py --config 3 >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kb$v=$? >> $S; done
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu"
timeout 300 $B > gpurun_out/plain_b1.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 150000 --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch.log 2>&1; echo ncul=$? >> $S
P="python scripts/prof_step.py --config 3 --steps 1"
timeout 300 $P > gpurun_out/plain_p.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg5_[AB]4 -s 4000 -c 2 -o gpurun_out/prof_cg_mom -f $P > gpurun_out/ncu_full.log 2>&1; echo ncuf=$? >> $S
