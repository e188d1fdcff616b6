#!/bin/bash
# Multi-GPU suite: parity via torchrun, then bench at N=$1 (c2 owner/contiguous, c3).
n=${1:-2}
out=gpurun_out/multi_n$n
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -x -q > $out/pytest_multi.log 2>&1; echo "pytest exit $?"; tail -3 $out/pytest_multi.log
run() {
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus $n "$@" 2> $out/bench_err.log | tail -1
}
run --config c2 > $out/bench_c2.json; echo "bench c2 exit $?"; cut -c1-300 $out/bench_c2.json
run --config c2 --assign contiguous > $out/bench_c2_contig.json; echo "bench c2 contiguous exit $?"
run --config c3 > $out/bench_c3.json; echo "bench c3 exit $?"
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 \
   bench.py --gpus $n --impl reference --steps 10 --warmup 3 > $out/bench_ref.json 2>> $out/bench_err.log; echo "ref exit $?"
