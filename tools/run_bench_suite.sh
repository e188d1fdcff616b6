#!/bin/bash
# Bench suite (1 GPU): GPU tests, smoke, the default bench line, the other
# configs and strategies, then the ncu launch list and one full capture of
# each hot kernel (collect, sample, two-level scan, fused update).
# usage: tools/run_bench_suite.sh <outdir>
out=gpurun_out/${1:-suite}
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -2 $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"
timeout 600 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench exit $?"
cut -c1-300 $out/bench_default.json
for c in c1 c3 c5; do
  timeout 900 python bench.py --config $c --cpu-budget 10 > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
timeout 600 python bench.py --strategy topk --no-cpu-baseline > $out/bench_c2_topk.json 2> $out/bench_c2_topk.err; echo "bench topk exit $?"
timeout 600 python bench.py --strategy fifo --no-cpu-baseline > $out/bench_c2_fifo.json 2> $out/bench_c2_fifo.err; echo "bench fifo exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err; echo "reference exit $?"
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
# the host-resident (PCIe-bound) collect of c3 (c5's 130 GB registered host
# table does not survive ncu's replay)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_tma -s 3 -c 1 \
    -o $out/collect_tma_c3_full python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
    > $out/ncu_full_collect_c3.log 2>&1
echo "full capture collect c3 exit $?"
