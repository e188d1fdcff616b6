#!/bin/bash
# c3 (4 KB host rows): the small-row TMA shape (chunk = row, 4 stages, the
# default since r01w) vs 3 / 2 stages of one row and the old 3 x 16 KB shape;
# headline (graph) and e2e traj/s.
out=gpurun_out/c3ab
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 200 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1; }
for rep in 1 2; do
  b > $out/auto_$rep.json
  GEAR_TMA_CHUNK=4096 GEAR_TMA_STAGES=3 b > $out/k4s3_$rep.json
  GEAR_TMA_CHUNK=4096 GEAR_TMA_STAGES=2 b > $out/k4s2_$rep.json
  GEAR_TMA_CHUNK=16384 GEAR_TMA_STAGES=3 b > $out/old_$rep.json
done
for f in $out/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', '%.3f M'%(d['value']/1e6), 'e2e %.3f M'%(d['e2e']['value']/1e6), 'eager %.3f M'%(d['graph']['eager_pipelined']['value']/1e6), 'frac=%.3f'%r['frac'], 'coll_ms=%.4f'%r['avg_launch_ms'])" 2>&1 | tail -1; done
