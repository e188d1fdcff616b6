"""Writer-path measurements (NEXT-1): gear_insert from device sources (device
plan + scatter + meta), and the split gear_allocate + gear_commit pair, eager
and captured in a CUDA graph.  CUDA events on the issuing stream; one JSON
line per case."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6538.6) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")) else 6538.6
s = torch.cuda.Stream()


def timed(fn, iters):
    for i in range(3):
        fn(i)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(iters):
        fn(i)
    e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / iters


for name, cap, B in (("c2", 100_000, 512), ("c1", 1024, 64), ("c1_4096", 100_000, 4096)):
    cfg = synth.CONFIGS["c2" if name == "c2" else "c1"]
    cols = [gear.Column(c.name, {"u8": gear.GEAR_U8, "i32": gear.GEAR_I32,
                                 "f32": gear.GEAR_F32}[c.dtype], tuple(c.shape), gear.GEAR_DEVICE)
            for c in cfg.cols]
    t = gear.Table(cap, cfg.seq_len, cols, None, max_batch=max(B, 4096))
    rbs = t.row_bytes
    src = [torch.randint(0, 255, (B, rb), dtype=torch.uint8, device="cuda") for rb in rbs]
    prio = torch.from_numpy(synth.priorities(B, seed=3)).cuda()
    out = torch.empty(B, dtype=torch.int64, device="cuda")

    def ins(i):
        gear.gear_insert(t.handle, 0, B, src, prio, out, s)

    ms = timed(ins, 20)
    payload = B * sum(rbs)
    print(json.dumps({"case": f"gear_insert {name}", "rows": B, "row_bytes": sum(rbs),
                      "us_per_call": round(ms * 1e3, 2), "rows_per_s": B / (ms / 1e3),
                      "hbm_gbs_read_plus_write": 2 * payload / (ms / 1e3) / 1e9,
                      "frac_of_hbm_copy_peak": 2 * payload / (ms / 1e3) / 1e9 / PEAK}), flush=True)

    def alloc_commit(i):
        gear.gear_allocate(t.handle, 0, B, out, s)
        gear.gear_commit(t.handle, 0, B, out, prio, s)

    ms_e = timed(alloc_commit, 50)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        alloc_commit(0)
    s.synchronize()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        for _ in range(10):
            alloc_commit(0)
    with torch.cuda.stream(s):
        ms_g = timed(lambda i: g.replay(), 10) / 10
    assert t.sync()[0] == 0
    print(json.dumps({"case": f"gear_allocate+gear_commit {name}", "rows": B,
                      "us_per_pair_eager": round(ms_e * 1e3, 2),
                      "us_per_pair_graph": round(ms_g * 1e3, 2),
                      "rows_per_s_graph": B / (ms_g / 1e3)}), flush=True)
    t.close()
