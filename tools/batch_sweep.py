"""Batch-size sweep of collection (the paper's E3: collection
throughput for B in {32 .. 1024}), on one GPU: for each config's table, B
trajectories are sampled with the config's strategy and collected; collect
time alone and the serial sample+collect step are timed with CUDA events
(median of 30 after 5 warm-ups).  One JSON line per (config, B).

usage: python tools/batch_sweep.py [c3 c5 c2 ...]   (default: c3 c5 c2)
Host tables are scaled to the box's RAM like bench.py (c5: GEAR_BENCH_HOST_FRAC)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

STRAT = {"prioritized": gear.GEAR_PRIORITIZED, "weighted": gear.GEAR_WEIGHTED,
         "uniform": gear.GEAR_UNIFORM, "fifo": gear.GEAR_FIFO, "lifo": gear.GEAR_LIFO}
BS = (32, 64, 128, 256, 512, 1024, 2048, 4096)

for name in (sys.argv[1:] or ["c3", "c5", "c2"]):
    cfg = synth.CONFIGS[name]
    cap, note = bench.scaled_capacity(cfg, 1)
    s = torch.cuda.Stream()
    t, _ = bench.build_table(cfg, None, 1, 0, cap, s)
    cols = list(range(len(t.row_bytes)))
    rb = sum(t.row_bytes)
    host = sum(synth.row_bytes(cfg, c) for c in cfg.cols if c.placement == "host")
    for B in BS:
        if B * rb > (8 << 30):
            continue
        idx = torch.empty(B, dtype=torch.int64, device="cuda")
        outs = [torch.empty((B, r), dtype=torch.uint8, device="cuda") for r in t.row_bytes]
        coll, step = [], []
        for i in range(35):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(s)
            gear.gear_sample(t.handle, STRAT[cfg.strategy], B, synth.SAMPLE_SEED_BASE + i, 0.4, idx,
                             None, None, None, s)
            e[1].record(s)
            gear.gear_collect(t.handle, B, idx, cols, outs, s)
            e[2].record(s)
            s.synchronize()
            if i >= 5:
                step.append(e[0].elapsed_time(e[2]))
                coll.append(e[1].elapsed_time(e[2]))
        assert t.sync()[0] == 0
        c_ms, s_ms = float(np.median(coll)), float(np.median(step))
        print(json.dumps({"config": name, "B": B, "row_bytes": rb, "host_row_bytes": host,
                          "collect_us": round(c_ms * 1e3, 2), "step_us": round(s_ms * 1e3, 2),
                          "collect_gbs": B * rb / (c_ms / 1e3) / 1e9,
                          "traj_per_s": B / (s_ms / 1e3), "capacity": cap,
                          **({"note": note} if note else {})}), flush=True)
    t.close()
