mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> $S
rm -f gpurun_out/kbench.jsonl
for v in base p5; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_1811_11842_b200/libch_b200_$v.so; fi
  for op in poisson mom_v; do CHB_LIB=$L timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo $v$op=$? >> $S; done
done
for d in 2 32; do CHB_DEFER=$d timeout 300 python scripts/kbench.py --solve poisson --config 2 | sed "s/^{/{\"lib\": \"defer$d\", /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done
