#!/bin/bash
# Multi-GPU suite: parity via torchrun, then bench at N=$1 for the configs.
n=${1:-2}
out=gpurun_out/multi_n$n
mkdir -p $out
{ nproc; free -g; df -h /dev/shm; nvidia-smi topo -m; } > $out/host.txt 2>&1
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
python -m pytest tests/test_gpu_multi.py -x -q > $out/pytest_multi.log 2>&1; echo "pytest exit $?"; tail -3 $out/pytest_multi.log
run() {
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus $n "$@" 2>> $out/bench_err.log | tail -1
}
run --config c2 > $out/bench_c2.json; echo "bench c2 exit $?"; cut -c1-200 $out/bench_c2.json
run --config c2 --assign contiguous > $out/bench_c2_contig.json; echo "bench c2 contiguous exit $?"
run --config c3 > $out/bench_c3.json; echo "bench c3 exit $?"
run --config c4 > $out/bench_c4.json; echo "bench c4 exit $?"
run --config c4 --strategy fifo > $out/bench_c4_fifo.json; echo "bench c4 fifo exit $?"
run --config c2 --strategy topk > $out/bench_c2_topk.json; echo "bench c2 topk exit $?"
run --config c2 --strategy fifo > $out/bench_c2_fifo.json; echo "bench c2 fifo exit $?"
run --config c5 > $out/bench_c5.json; echo "bench c5 exit $?"
run --impl reference --steps 3 --warmup 3 > $out/bench_reference.json; echo "reference exit $?"
