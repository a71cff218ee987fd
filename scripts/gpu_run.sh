mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
rm -f gpurun_out/kbench.jsonl
for s in poisson mom_v; do timeout 300 python scripts/kbench.py --solve $s >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo kb_$s=$? >> $S; done
timeout 300 python scripts/kbench.py --solve poisson --config 2 >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err
L=$PWD/paper_1811_11842_b200/libch_b200_trace.so
rm -f gpurun_out/trace.jsonl
CHB_LIB=$L timeout 300 python scripts/trace_sweep.py --solve poisson --config 3 --nb 740 >> gpurun_out/trace.jsonl 2>> gpurun_out/trace.err; echo t1=$? >> $S
