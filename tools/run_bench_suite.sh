#!/bin/bash
# Bench suite (1 GPU): parity tests, the default bench line, the other configs,
# then the ncu launch list and one full capture of the collect kernel.
# usage: tools/run_bench_suite.sh <outdir>
out=gpurun_out/${1:-suite}
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
python -m pytest tests -m gpu -x -q > $out/pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -2 $out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"
python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench exit $?"
cat $out/bench_default.json | cut -c1-400
for c in c1 c3 c5; do
  python bench.py --config $c --cpu-budget 10 > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $out/plain_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'collect|sample_kernel|scan_kernel|quantize_kernel|tag_kernel|apply_kernel|fused_kernel' -c 80 \
    --csv --log-file $out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    > $out/ncu_launches.log 2>&1
echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k regex:collect_tma -s 3 -c 1 \
    -o $out/collect_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    > $out/ncu_full.log 2>&1
echo "full capture exit $?"
