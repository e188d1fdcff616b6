"""Full rebuilds of the two-level CDF (scan2_kernel) on a large table, for ncu:
every iteration re-selects cdf_levels=2, which forgets both buffers' builds."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000_000
t = gear.Table(N, 1, [gear.Column("x", gear.GEAR_U8, (16,))], None, max_batch=4096)
s = torch.cuda.Stream()
rows = torch.zeros((1 << 20, 16), dtype=torch.uint8, device="cuda")
prio = synth.priorities(N, seed=1, zero_frac=0.01)
for k0 in range(0, N, 1 << 20):
    m = min(1 << 20, N - k0)
    gear.gear_insert(t.handle, 0, m, [rows], prio[k0:k0 + m], None, s)
idx = torch.zeros(512, dtype=torch.int64, device="cuda")
times = []
for i in range(6):
    gear.gear_table_set_tuning(t.handle, "cdf_levels", 2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    gear.gear_sample(t.handle, gear.GEAR_PRIORITIZED, 512, i, 0.4, idx, None, None, None, s)
    e1.record(s)
    s.synchronize()
    times.append(e0.elapsed_time(e1))
assert t.sync()[0] == 0
t.close()
print("full rebuild + sample ms:", [round(x, 4) for x in times])
