"""CDF rebuild throughput at N keys (one shard): the flat decoupled look-back
scan (cdf_levels 1: every sample after a key write rebuilds the whole CDF) and
a full two-level rebuild (cdf_levels 2 re-selected: both buffers forgotten).
Rebuild time = (update of 1 key + sample of 1 draw) - (update + sample without
rebuild is impossible, so: sample right after a layout switch minus a sample
with a clean CDF); CUDA events, median of 20.  Run under ncu for kernel
durations and DRAM bytes:  python tools/scan_bench.py 40000000 [reps] [variants]
(variants: comma list of levels1_tile, levels1_chunk, levels2).  Also times a
device copy of the same bytes (the size-matched streaming ceiling)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
t = gear.Table(N, 1, [gear.Column("x", gear.GEAR_U8, (16,))], None, max_batch=4096)
s = torch.cuda.Stream()
rows = torch.zeros((1 << 20, 16), dtype=torch.uint8, device="cuda")
prio = synth.priorities(N, seed=1, zero_frac=0.01)
for k0 in range(0, N, 1 << 20):
    m = min(1 << 20, N - k0)
    gear.gear_insert(t.handle, 0, m, [rows], prio[k0:k0 + m], None, s)
idx = torch.zeros(1, dtype=torch.int64, device="cuda")
p1 = torch.ones(1, dtype=torch.float64, device="cuda")


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    fn()
    e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1)


def sample():
    gear.gear_sample(t.handle, gear.GEAR_PRIORITIZED, 1, 5, 0.4, idx, None, None, None, s)


out = {"keys": N, "bytes_per_rebuild": 16 * N}
variants = [("levels1_tile", 1, 0), ("levels1_chunk", 1, 1), ("levels2", 2, -1)]
if len(sys.argv) > 3:
    variants = [v for v in variants if v[0] in sys.argv[3].split(",")]
for name, levels, chunk in variants:
    gear.gear_table_set_tuning(t.handle, "cdf_levels", levels)
    gear.gear_table_set_tuning(t.handle, "scan_chunk", chunk)
    sample()
    base, full = [], []
    for i in range(reps):
        if levels == 1:
            base.append(timed(sample))                  # clean CDF: no rebuild
            gear.gear_update_priorities(t.handle, 1, idx, p1, gear.GEAR_F64, None, s)
            full.append(timed(sample))                  # rebuilds the whole CDF
        else:
            gear.gear_table_set_tuning(t.handle, "cdf_levels", 2)   # forget both builds
            full.append(timed(sample))                  # full rebuild of one buffer
            sample()                                    # ... and of the other
            base.append(timed(sample))                  # both built: every tile clean
    ms = float(np.median(full) - np.median(base))
    out[name] = {"rebuild_us": ms * 1e3, "GBps": 16 * N / (ms / 1e3) / 1e9,
                 "frac_of_6456": 16 * N / (ms / 1e3) / 1e9 / 6456.2}
# size-matched copy: the same bytes (N u64 read + N u64 written) as one
# device-to-device copy, the ceiling a streaming kernel of this size reaches
a = torch.empty(N, dtype=torch.int64, device="cuda")
b = torch.empty_like(a)
with torch.cuda.stream(s):
    cp = [timed(lambda: b.copy_(a)) for _ in range(reps)]
ms = float(np.median(cp))
out["copy_same_bytes"] = {"us": ms * 1e3, "GBps": 16 * N / (ms / 1e3) / 1e9}
assert t.sync()[0] == 0
t.close()
print(json.dumps(out))
