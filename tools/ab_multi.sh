#!/bin/bash
# A/B of library variants on the N-GPU bench: tools/ab_multi.sh N outdir "bench args" lib1 lib2 ...
# (lib "default" = the in-tree libgear.so)
n=$1; out=gpurun_out/$2; args=$3; shift 3
mkdir -p $out
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
for lib in "$@"; do
  if [ "$lib" = default ]; then L=paper_2310_05205_b200/libgear.so; else L=paper_2310_05205_b200/ab/libgear_$lib.so; fi
  GEAR_LIB=$L timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
     --master-port 29517 bench.py --gpus $n $args 2>> $out/err_$lib.log | tail -1 > $out/bench_$lib.json
  python - $out/bench_$lib.json $lib <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(sys.argv[2], "value %.3fM" % (d["value"] / 1e6), "ms %.4f" % d["ms_per_step"], "coll %.4f" % r["avg_launch_ms"],
          "frac %.3f" % r["frac"], "sel_only %.4f" % d["selection"]["only_ms_per_step"], "e2e %.3fM" % (d["e2e"]["value"] / 1e6))
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
done
