#!/bin/bash
# Round-2 (late) check: build, the chunked look-back scan's parity and timing
# (event-timed rebuilds + ncu kernel durations / DRAM bytes at 5-40 M keys),
# then the whole GPU suite, smoke and the default bench line.
out=gpurun_out/${1:-r02t}
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_stress.py -q -x > $out/pytest_scan.log 2>&1; echo "pytest scan exit $?"; tail -2 $out/pytest_scan.log
for n in 5000000 10000000 20000000 40000000; do
  timeout 300 python tools/scan_bench.py $n 20 > $out/scan_$n.json 2>&1; echo "scan $n $?"; cat $out/scan_$n.json
done
for n in 10000000 40000000; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:scan --csv --log-file $out/ncu_scan_$n.csv \
    python tools/scan_bench.py $n 5 > $out/ncu_scan_$n.log 2>&1; echo "ncu scan $n $?"
done
[ -n "$QUICK" ] && exit 0
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $out/pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -2 $out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench exit $?"
python tools/summarize_bench.py $out
