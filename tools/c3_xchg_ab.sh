#!/bin/bash
# c3 at N GPUs: mailbox exchanges (default) vs NCCL all-gathers, serial vs pipelined collect
n=${1:-4}
python __graft_entry__.py > /dev/null 2>&1
for v in "GEAR_PEER_XCHG=1" "GEAR_PEER_XCHG=0"; do
 for a in owner contiguous; do
  env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $n --config c3 --assign $a --no-cpu-baseline --steps 300 2>/dev/null | tail -1 | \
    python3 -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$v $a]', round(d['value']/1e6,3), 'coll', round(r['avg_launch_ms'],4), 'serial', round(d['serial']['ms_per_step'],4), round(d['serial']['collect_avg_ms'],4), 'sel', round(d['selection']['only_ms_per_step'],4), round(d['selection']['sample_only_ms'],4))"
 done
done
