mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
for c in 0 1 2; do CHB_PERSIST=1 timeout 900 python bench.py --config $c --no-cpu > gpurun_out/bench_p_c$c.log 2>&1; echo bench_p_c$c=$? >> $S; done
