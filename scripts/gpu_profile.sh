#!/bin/sh
# One gpurun call: the headline bench, two windows of its launch list (1 step,
# serialised) and ncu --set full captures of the top kernels (each after a
# plain run of the same command).  Reports are written to /tmp/prof on the box
# and summarised there (scripts/ncu_summary.py): only the summaries and the
# smallest reports come back in gpurun_out/ (64 MiB cap).
mkdir -p gpurun_out /tmp/prof
S=gpurun_out/status.txt; : > $S
if [ "${SKIP_BENCH:-0}" = 0 ]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$? >> $S
fi
B1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --matvec 0"
timeout 300 $B1 > gpurun_out/plain_b1.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file /tmp/prof/launches_head.csv $B1 > gpurun_out/ncu_l1.log 2>&1; echo launches=$? >> $S
for op in mom_v poisson; do
  timeout 300 python scripts/kbench.py --solve $op > gpurun_out/plain_$op.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_iter -s 300 -c 2 \
      -o /tmp/prof/prof_$op python scripts/kbench.py --solve $op > gpurun_out/ncu_$op.log 2>&1
  echo ncu_$op=$? >> $S
done
timeout 300 python scripts/kbench.py --solve poisson > gpurun_out/plain_px.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cgs_px -s 20 -c 1 \
    -o /tmp/prof/prof_px python scripts/kbench.py --solve poisson > gpurun_out/ncu_px.log 2>&1
echo ncu_px=$? >> $S
K1="python scripts/kbench.py --steps 1 --warmup 0"
timeout 300 $K1 > gpurun_out/plain_k1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ch_rm -s 20 -c 1 \
    -o /tmp/prof/prof_ch $K1 > gpurun_out/ncu_ch.log 2>&1
echo ncu_ch=$? >> $S
ls -la /tmp/prof > gpurun_out/prof_ls.txt
ARGS=""
for r in /tmp/prof/*.ncu-rep; do ARGS="$ARGS --rep $r"; done
for l in /tmp/prof/launches_*.csv; do ARGS="$ARGS --launches $l"; done
[ -f gpurun_out/bench.json ] && ARGS="$ARGS --bench gpurun_out/bench.json"
python scripts/ncu_summary.py $ARGS --out gpurun_out/r02 > gpurun_out/summary.log 2>&1
echo summary=$? >> $S
cp profiles/traffic.json gpurun_out/traffic.json 2>/dev/null
# bring back the reports that fit (largest first skipped)
for r in /tmp/prof/prof_mom_v.ncu-rep /tmp/prof/prof_poisson.ncu-rep; do
  sz=$(stat -c %s $r 2>/dev/null || echo 0)
  [ "$sz" -lt 20000000 ] && cp $r gpurun_out/
done
# the launch list itself (5000 launches, ~1 MB)
cp /tmp/prof/launches_head.csv gpurun_out/ 2>/dev/null
du -sh gpurun_out >> $S
