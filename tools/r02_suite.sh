#!/bin/bash
# Round-2 1-GPU suite: build, GPU tests, smoke, every config's bench line, the
# reference arm, the ncu launch list (+ NVTX ranges) and full captures of the
# hot kernels.  usage: tools/r02_suite.sh <outdir>
out=gpurun_out/${1:-r02s}
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --durations=25 > $out/pytest_gpu.log 2>&1; echo "pytest gpu exit $?"; tail -2 $out/pytest_gpu.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke exit $?"
fi
timeout 900 python bench.py > $out/bench_default.json 2> $out/bench_default.err; echo "bench exit $?"
for c in c1 c3 c4 c5; do
  timeout 1200 python bench.py --config $c --cpu-budget 10 > $out/bench_$c.json 2> $out/bench_$c.err; echo "bench $c exit $?"
done
for st in topk fifo; do
  timeout 900 python bench.py --strategy $st --no-cpu-baseline > $out/bench_c2_$st.json 2> $out/bench_c2_$st.err; echo "bench $st exit $?"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err; echo "reference exit $?"
# ncu: launch list of the default bench (eager, small K), with NVTX ranges
K='collect|sample_kernel|scan2_kernel|scan_kernel|assign_kernel|fused_kernel|alpha_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --nvtx -k regex:"$K" -c 60 --csv --print-nvtx-rename kernel \
    --log-file $out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
    > $out/ncu_launches.log 2>&1
echo "launch list exit $?"
timeout 900 ncu --nvtx --nvtx-include "gear_sample/" --metrics gpu__time_duration.sum --clock-control none -c 12 --csv \
    --log-file $out/nvtx_gear_sample.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
    > $out/ncu_nvtx.log 2>&1
echo "nvtx filter exit $?"
for kern in collect_tma sample_kernel scan2_kernel fused_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kern -s 3 -c 1 \
      -o $out/${kern}_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
      > $out/ncu_full_$kern.log 2>&1
  echo "full capture $kern exit $?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:collect_tma -s 3 -c 1 \
    -o $out/collect_tma_c3_full python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --graph 0 \
    > $out/ncu_full_collect_c3.log 2>&1
echo "full capture collect c3 exit $?"
python tools/summarize_bench.py $out
