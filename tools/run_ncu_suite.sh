#!/bin/bash
# The ncu part of run_bench_suite.sh alone (launch list + full captures).
# usage: tools/run_ncu_suite.sh <outdir>
out=gpurun_out/${1:-suite}
mkdir -p $out
K='collect|sample_kernel|scan2_kernel|scan_kernel|assign_kernel|fused_kernel|alpha_kernel'
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 > $out/plain_small.log 2>&1 &&
# (the table fill's row copies run as insert_rows_* kernels: not matched)
FILL=${FILL:-0}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"$K" -s $FILL -c 80 \
    --csv --log-file $out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
    > $out/ncu_launches.log 2>&1
echo "launch list exit $?"
for kern in collect_tma sample_kernel scan2_kernel fused_kernel; do
  skip=3; [ $kern = collect_tma ] && skip=$((FILL + 3))
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s $skip -c 1 \
      -o $out/${kern}_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
      > $out/ncu_full_$kern.log 2>&1
  echo "full capture $kern exit $?"
done
