#!/bin/bash
# c2 contiguous-slice collect (half / 3 quarters of the rows over NVLink) under
# collect-kernel shapes: tools/contig_sweep.sh N
n=${1:-2}
python __graft_entry__.py > /dev/null 2>&1
for v in "" "GEAR_COLLECT_PEER_LSU=1" "GEAR_TMA_STAGES=6 GEAR_TMA_CTAS=1" "GEAR_TMA_CHUNK=32768 GEAR_TMA_STAGES=3 GEAR_TMA_CTAS=2" "GEAR_TMA_CHUNK=8192 GEAR_TMA_STAGES=6 GEAR_TMA_CTAS=2" "GEAR_TMA_CHUNK=8192 GEAR_TMA_STAGES=4 GEAR_TMA_CTAS=4"; do
  env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $n --config c2 --assign contiguous --no-cpu-baseline --steps 300 2>/dev/null | tail -1 | \
    python3 -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('[$v]', round(d['value']/1e6,3), 'coll', round(r['avg_launch_ms'],4), r['bound'], 'frac', round(r['frac'],3), 'nvl_probe', round(r['probes']['nvlink_pull_GBps'],1), 'remote', round(r['remote_fraction'],3))"
done
