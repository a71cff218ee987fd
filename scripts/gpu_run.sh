mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo bench=$? >> $S
rm -f gpurun_out/kbench.jsonl
for s in poisson mom_u mom_v; do timeout 300 python scripts/kbench.py --solve $s >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kb_$s=$? >> $S; done
timeout 300 python scripts/kbench.py --solve poisson --config 2 >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err
for c in 0 1 2; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/bench_c$c.log 2>&1; echo bench_c$c=$? >> $S; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo launches=$? >> $S
V="python scripts/kbench.py --solve mom_v"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 3000 -c 2 -o gpurun_out/prof_cgs_v -f $V > gpurun_out/ncu_full_v.log 2>&1; echo ncufv=$? >> $S
P="python scripts/kbench.py --solve poisson"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 3000 -c 2 -o gpurun_out/prof_cgs_p -f $P > gpurun_out/ncu_full_p.log 2>&1; echo ncufp=$? >> $S
timeout 900 ncu --set full --clock-control none -k regex:k_cgs_px -s 50 -c 1 -o gpurun_out/prof_px -f $P > gpurun_out/ncu_px.log 2>&1; echo ncupx=$? >> $S
du -sh gpurun_out >> $S
