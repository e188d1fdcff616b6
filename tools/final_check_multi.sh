#!/bin/bash
# Final multi-GPU check at N=$1: multi-rank parity, then the driver's default
# bench command (no config flags) and the reference arm under torchrun.
n=${1:-2}
out=gpurun_out/r01x_n$n
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $out/pytest_multi.log 2>&1; echo "pytest exit $?"; tail -2 $out/pytest_multi.log
for impl in ours reference; do
  extra=""; [ $impl = reference ] && extra="--impl reference --steps 3 --warmup 3"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 \
     bench.py --gpus $n $extra > $out/bench_$impl.json 2> $out/bench_$impl.err
  echo "bench $impl exit $?"; tail -1 $out/bench_$impl.json | cut -c1-300
done
