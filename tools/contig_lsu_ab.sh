#!/bin/bash
# c2 contiguous-slice collect at N ranks: TMA bulk pipeline (default) vs the
# all-LSU collect kernel (16-B loads, 8 in flight per lane) for every row.
n=${1:-2}
out=gpurun_out/${2:-contig_lsu_n$n}
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
for v in "" "GEAR_COLLECT_IMPL=lsu" "GEAR_COLLECT_IMPL=lsu GEAR_COLLECT_CHUNK=32768" "GEAR_COLLECT_IMPL=lsu GEAR_COLLECT_CHUNK=4096"; do
  for a in contiguous owner; do
  env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus $n --config c2 --assign $a --no-cpu-baseline --steps 300 2>>$out/err.log | tail -1 > $out/tmp.json
  python3 -c "import json,sys; d=json.load(open('$out/tmp.json')); r=d['roofline']; print('[$v] $a', round(d['value']/1e6,3), 'e2e', round(d['e2e']['value']/1e6,3), 'coll', round(r['avg_launch_ms'],4), r['bound'], 'frac', round(r['frac'],3), 'nvl_probe', round(r['probes']['nvlink_pull_GBps'],1), 'remote', round(r['remote_fraction'],3))" | tee -a $out/sweep.txt
  done
done
