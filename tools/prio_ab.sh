for n in 4; do
for a in "--collect-priority normal" "--collect-priority high"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $n --config c2 --strategy topk --no-cpu-baseline --steps 500 $a 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$a topk', round(d['value']/1e6,3), round(r['avg_launch_ms'],4), round(r['frac'],3))"
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $n --config c2 --no-cpu-baseline --steps 500 $a 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$a c2', round(d['value']/1e6,3), round(r['avg_launch_ms'],4), round(r['frac'],3))"
done; done
