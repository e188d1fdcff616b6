#!/bin/bash
# Why do host-resident configs lose PCIe efficiency at N>1?  c5 variants at N=$1.
n=${1:-4}
out=gpurun_out/host_multi_n$n
mkdir -p $out
python __graft_entry__.py > /dev/null 2>&1
run() {
  tag=$1; shift
  env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
     --master-port 29511 bench.py --gpus $n --config c5 --steps 10 --warmup 3 $BENCH_ARGS 2>> $out/err.log | tail -1 > $out/$tag.json
  python -c "
import json; d=json.load(open('$out/$tag.json')); r=d['roofline']
print('$tag', d['config']['capacity'], 'frac=%.3f'%r['frac'], 'coll_ms=%.3f'%r['avg_launch_ms'], 'remote=%.3f'%r['remote_fraction'])"
}
run default X=1
run lsu GEAR_COLLECT_IMPL=lsu
BENCH_ARGS="--assign contiguous" run contiguous X=1
GEAR_SMALL=1 run small GEAR_BENCH_HOST_FRAC=0.05
