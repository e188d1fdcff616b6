"""Flat (decoupled look-back) vs two-level incremental CDF: time of one
update + sample (which rebuilds the CDF) per iteration, CUDA events, for a
few table sizes and update sizes.  Prints one JSON line per case."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

ITERS = 50
s = torch.cuda.Stream()
for N in (100_000, 1_000_000, 10_000_000, 40_000_000):
    t = gear.Table(N, 1, [gear.Column("x", gear.GEAR_U8, (16,))], None, max_batch=8192)
    rows = torch.zeros((1 << 20, 16), dtype=torch.uint8, device="cuda")
    prio = synth.priorities(N, seed=1, zero_frac=0.01)
    for k0 in range(0, N, 1 << 20):
        m = min(1 << 20, N - k0)
        gear.gear_insert(t.handle, 0, m, [rows], prio[k0:k0 + m], None, s)
    rng = np.random.default_rng(0)
    out = torch.empty(512, dtype=torch.int64, device="cuda")
    for B in (16, 512, 8192):
        ids = [torch.from_numpy(rng.integers(0, N, B).astype(np.int64)).cuda() for _ in range(4)]
        pr = [torch.from_numpy(synth.priorities(B, seed=k)).cuda() for k in range(4)]
        for levels in (1, 2):
            gear.gear_table_set_tuning(t.handle, "cdf_levels", levels)
            res = {}
            for mode in ("update+sample", "sample only"):
                def it(i):
                    if mode == "update+sample":
                        gear.gear_update_priorities(t.handle, B, ids[i % 4], pr[i % 4],
                                                    gear.GEAR_F64, None, s)
                    gear.gear_sample(t.handle, gear.GEAR_PRIORITIZED, 512, i, 0.4, out, None,
                                     None, None, s)
                for i in range(5):
                    it(i)
                s.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for i in range(ITERS):
                    it(i)
                e1.record(s)
                s.synchronize()
                res[mode] = e0.elapsed_time(e1) / ITERS * 1e3
            assert t.sync()[0] == 0
            print(json.dumps({"N": N, "B_update": B, "cdf_levels": levels,
                              "us_update_sample": round(res["update+sample"], 2),
                              "us_sample_only": round(res["sample only"], 2),
                              "us_rebuild_and_update": round(res["update+sample"]
                                                             - res["sample only"], 2)}),
                  flush=True)
    t.close()
