#!/bin/bash
# Can consecutive host (PCIe) collects overlap their ramp-up / drain?  c3 at
# N=1: default vs two collect streams, with and without stages small enough
# (GEAR_TMA_CHUNK=4096) that the next collect's CTAs fit beside the current one's.
out=gpurun_out/c3ov
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() {  # name env... -- bench args
  local name=$1; shift
  env "$@" timeout 200 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 > $out/$name.json
}
for rep in 1 2; do
  run A$rep X=1
  env timeout 200 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --collect-streams 2 2>/dev/null | tail -1 > $out/B$rep.json
  GEAR_TMA_CHUNK=4096 GEAR_TMA_STAGES=4 timeout 200 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --collect-streams 2 2>/dev/null | tail -1 > $out/C$rep.json
  GEAR_TMA_CHUNK=4096 GEAR_TMA_STAGES=4 GEAR_TMA_CTAS=1 timeout 200 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --collect-streams 2 2>/dev/null | tail -1 > $out/D$rep.json
  GEAR_TMA_CHUNK=4096 GEAR_TMA_STAGES=4 timeout 200 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1 > $out/E$rep.json
  GEAR_TMA_CHUNK=4096 GEAR_TMA_STAGES=8 GEAR_TMA_CTAS=1 timeout 200 python bench.py --config c3 --steps 100 --warmup 10 --no-cpu-baseline --collect-streams 2 2>/dev/null | tail -1 > $out/F$rep.json
done
for f in $out/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; g=d.get('graph',{}); print('$f', '%.2f M'%(d['value']/1e6), 'frac=%.3f'%r['frac'], 'step_frac=%.3f'%r['step_frac'], 'coll_ms=%.4f'%r['avg_launch_ms'], 'eager=%.2f M'%(g.get('eager_pipelined',{}).get('value',0)/1e6))" 2>&1 | tail -1; done
