#!/bin/bash
# Final 1-GPU check of the last code: GPU tests, smoke, default bench line, and
# the CDF rebuild benchmark (flat per-tile / chunked look-back, two-level) at
# 5-40 M keys with ncu kernel durations.
out=gpurun_out/${1:-r02f}
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > $out/pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -2 $out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench exit $?"
for n in 5000000 10000000 20000000 40000000; do
  timeout 300 python tools/scan_bench.py $n 20 > $out/scan_$n.json 2>&1; echo "scan $n $(cat $out/scan_$n.json)"
done
for n in 10000000 40000000; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:scan --csv --log-file $out/ncu_scan_$n.csv python tools/scan_bench.py $n 5 > /dev/null 2>&1; echo "ncu scan $n $?"
done
python tools/summarize_bench.py $out
