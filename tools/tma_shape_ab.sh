#!/bin/bash
# A/B of the TMA collect shape in the full pipelined step (not the collect
# alone): default 2 CTAs x 3 stages x 16 KB vs shapes with less shared memory
# per SM, which leave room for the next step's sample kernel beside the collect.
# Usage: tools/tma_shape_ab.sh <config> [steps]
cfg=${1:-c2}; steps=${2:-100}
out=gpurun_out/tma_ab_$cfg
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
b() { timeout 300 python bench.py --config $cfg --steps $steps --warmup 10 --no-cpu-baseline 2>/dev/null | tail -1; }
for rep in 1 2; do
  b > $out/def_$rep.json
  GEAR_TMA_STAGES=2 b > $out/s2_$rep.json
  GEAR_TMA_CTAS=1 GEAR_TMA_STAGES=4 b > $out/c1s4_$rep.json
  GEAR_TMA_CTAS=4 GEAR_TMA_STAGES=2 GEAR_TMA_CHUNK=8192 b > $out/c4s2k8_$rep.json
done
for f in $out/*.json; do python -c "
import json; d=json.load(open('$f')); r=d['roofline']; print('$f', '%.3f M'%(d['value']/1e6), 'frac=%.3f'%r['frac'], 'step_frac=%.3f'%r['step_frac'], 'coll_ms=%.4f'%r['avg_launch_ms'])" 2>&1 | tail -1; done
