#!/bin/bash
# Round-1 measurement: plain bench (c2, N=1), then the ncu launch list and one
# full capture of the collect kernel of the same command.
set -o pipefail
mkdir -p gpurun_out/r01
python __graft_entry__.py > gpurun_out/r01/build.log 2>&1 || exit 3
python bench.py --steps 50 --warmup 5 > gpurun_out/r01/bench_c2.json 2> gpurun_out/r01/bench_c2.err || exit 4
cat gpurun_out/r01/bench_c2.json
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01/plain_small.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:'collect_kernel|sample_kernel|scan_kernel|quantize_kernel|tag_kernel|apply_kernel' -c 60 \
    --csv --log-file gpurun_out/r01/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r01/ncu_launches.log 2>&1
echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k regex:collect_kernel -s 3 -c 1 \
    -o gpurun_out/r01/collect_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/r01/ncu_full.log 2>&1
echo "full capture exit $?"
