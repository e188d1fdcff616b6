#!/bin/bash
# Bench suite (1 GPU): GPU tests, smoke, the default bench line, the other
# configs, then the ncu launch list and one full capture of the collect kernel.
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
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 > $out/plain_small.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'collect|sample_kernel|scan_kernel|assign_kernel|fused_kernel' -c 80 \
    --csv --log-file $out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
    > $out/ncu_launches.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_tma -s 3 -c 1 \
    -o $out/collect_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
    > $out/ncu_full.log 2>&1
echo "full capture exit $?"
