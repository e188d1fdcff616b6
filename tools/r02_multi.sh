#!/bin/bash
# Round-2 multi-GPU measurement: parity (NCCL and shared-device), then bench
# lines at N=$1 (both assignments are in every line), c2 / c3 / c2 TopK.
n=${1:-2}
out=gpurun_out/${2:-r02_n$n}
mkdir -p $out
{ nproc; free -g; nvidia-smi topo -m; } > $out/host.txt 2>&1
python __graft_entry__.py > $out/build.log 2>&1 || exit 3
[ -z "$SKIP_TESTS" ] && { timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > $out/pytest_multi.log 2>&1; echo "pytest multi exit $?"; tail -2 $out/pytest_multi.log; }
run() {
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 \
     bench.py --gpus $n "$@" 2>> $out/bench_err.log | tail -1
}
run --config c2 > $out/bench_c2.json; echo "bench c2 exit $?"
run --config c3 > $out/bench_c3.json; echo "bench c3 exit $?"
run --config c2 --strategy topk --no-cpu-baseline > $out/bench_c2_topk.json; echo "bench c2 topk exit $?"
python - <<'PY' $out
import json, sys, glob
for f in sorted(glob.glob(sys.argv[1] + "/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unparsable", e); continue
    r = d["roofline"]
    print(f.split("/")[-1], "value %.3fM" % (d["value"] / 1e6), "ms %.4f" % d["ms_per_step"],
          "e2e %.3fM" % (d["e2e"]["value"] / 1e6), r["bound"], "frac %.3f" % r["frac"],
          "step_frac %.3f" % r.get("step_frac", 0), "remote %.3f" % r.get("remote_fraction", 0),
          "peak %.1f" % r["peak"], "sel_only_ms %.4f" % d["selection"]["only_ms_per_step"], "coll_ms %.4f" % r["avg_launch_ms"],
          {k: round(v["value"] / 1e6, 3) for k, v in d.get("assignments", {}).items()})
PY
