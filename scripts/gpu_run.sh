# build-variant experiment: ring depth x register budget
mkdir -p gpurun_out
S=gpurun_out/status.txt; : > $S
rm -f gpurun_out/kbench.jsonl
for v in base mb65 n8m8 n12m6; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_1811_11842_b200/libch_b200_$v.so; fi
  for op in poisson mom_v; do CHB_LIB=$L timeout 300 python scripts/kbench.py --solve $op | sed "s/^{/{\"lib\": \"$v\", /" >> gpurun_out/kbench.jsonl 2>> gpurun_out/kbench.err; done
done
echo done >> $S
