#!/bin/bash
# A/B of environment settings on the bench: tools/env_ab.sh N "bench args" "ENV1=a ENV2=b" "ENV1=c" ...
# (N = 1: plain python; N > 1: torchrun)
n=$1; args=$2; shift 2
python __graft_entry__.py > /dev/null 2>&1
for v in "$@"; do
  if [ "$n" = 1 ]; then
    out=$(env $v timeout 900 python bench.py $args 2>/dev/null | tail -1)
  else
    out=$(env $v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
          --master-port 29517 bench.py --gpus $n $args 2>/dev/null | tail -1)
  fi
  echo "$out" | python3 -c "import json,sys
try:
    d=json.loads(sys.stdin.read()); r=d['roofline']
    print('N=$n [$v] $args', '%.3fM' % (d['value']/1e6), 'coll %.4f' % r['avg_launch_ms'], r['bound'], 'frac %.3f' % r['frac'], 'e2e %.3fM' % (d['e2e']['value']/1e6), {k: round(x['value']/1e6,3) for k,x in d.get('assignments',{}).items()})
except Exception as e:
    print('N=$n [$v] failed', e)"
done
