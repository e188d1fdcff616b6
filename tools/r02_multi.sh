#!/bin/bash
# Round-2 multi-GPU measurement: parity (NCCL and shared-device), then bench
# lines at N=$1 (both assignments are in every line), c2 / c3 / c2 TopK.
n=${1:-2}
out=gpurun_out/${2:-r02_n$n}
mkdir -p $out
{ nproc; free -g; nvidia-smi topo -m; } > $out/host.txt 2>&1
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
[ -z "$SKIP_TESTS" ] && { timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > $out/pytest_multi.log 2>&1; echo "pytest multi exit $?"; tail -2 $out/pytest_multi.log; }
run() {
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus $n "$@" 2>> $out/bench_err.log | tail -1
}
run --config c2 > $out/bench_c2.json; echo "bench c2 exit $?"
run --config c3 > $out/bench_c3.json; echo "bench c3 exit $?"
run --config c2 --strategy topk --no-cpu-baseline > $out/bench_c2_topk.json; echo "bench c2 topk exit $?"
run --config c2 --strategy fifo --no-cpu-baseline > $out/bench_c2_fifo.json; echo "bench c2 fifo exit $?"
[ -n "$WITH_HOST" ] && { run --config c4 --no-cpu-baseline --steps 200 > $out/bench_c4.json; echo "bench c4 exit $?";
  run --config c5 --no-cpu-baseline --steps 100 > $out/bench_c5.json; echo "bench c5 exit $?"; }
run --impl reference --steps 3 --warmup 3 > $out/bench_reference.json; echo "reference exit $?"
python tools/summarize_bench.py $out
