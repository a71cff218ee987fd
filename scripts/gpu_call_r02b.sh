mkdir -p gpurun_out; S=gpurun_out/status.txt; : > $S
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
for v in "" _w288 _w544; do for op in mom_v poisson; do CHB_LIB=$PWD/paper_1811_11842_b200/libch_b200$v.so timeout 300 python scripts/kbench.py --solve $op --stride 1 > gpurun_out/kbw_${op}$v.json 2>&1; done; done
for ny in 2048 1024 512; do for op in mom_v poisson; do timeout 300 python scripts/kbench.py --solve $op --nx 4096 --ny $ny --stride 1 > gpurun_out/kbslab_${op}_$ny.json 2>&1; done; done
timeout 1500 python scripts/diag_steps.py --n 16384 --steps 2 > gpurun_out/diag_16384.jsonl 2>&1; echo diag16k=$? >> $S
