mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
for v in base c24 c48 c64 base; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_1811_11842_b200/libch_b200_$v.so; fi
  for op in poisson; do CHB_LIB=$L timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; echo $v$op=$? >> $S; done
done
