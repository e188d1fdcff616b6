"""Host-side cost of each C-ABI call (development tool): mean wall time of
1000 back-to-back calls with no synchronisation (the GPU queue absorbs the
work), on a c1 table."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

cfg = synth.CONFIGS["c1"]
dt = {"u8": gear.GEAR_U8, "i32": gear.GEAR_I32, "f32": gear.GEAR_F32}
t = gear.Table(cfg.capacity, cfg.seq_len, [gear.Column(c.name, dt[c.dtype], c.shape) for c in cfg.cols])
s = torch.cuda.Stream()
rows = [torch.zeros((cfg.capacity, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
gear.gear_insert(t.handle, 0, cfg.capacity, rows, synth.priorities(cfg.capacity), None, s)
B = 64
idx = torch.zeros(B, dtype=torch.int64, device="cuda")
w = torch.empty(B, dtype=torch.float32, device="cuda")
p = torch.ones(B, dtype=torch.float64, device="cuda")
outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
h = t.handle
sid = s.cuda_stream
L = gear.load()
calls = {
    "gear_sample(prioritized)": lambda: L.gear_sample(h, gear.GEAR_PRIORITIZED, B, 1, 0.4, idx.data_ptr(), w.data_ptr(), None, None, sid),
    "gear_collect(3 cols)": lambda: gear.gear_collect(h, B, idx, [0, 1, 2], outs, sid),
    "gear_update_priorities": lambda: L.gear_update_priorities(h, B, idx.data_ptr(), p.data_ptr(), gear.GEAR_F64, None, sid),
    "binding gear_sample": lambda: gear.gear_sample(h, gear.GEAR_PRIORITIZED, B, 1, 0.4, idx, w, None, None, s),
    "torch empty launch (reference)": lambda: torch.cuda._sleep(0),
}
for name, fn in calls.items():
    for _ in range(50):
        fn()
    s.synchronize()
    t0 = time.perf_counter()
    for _ in range(1000):
        fn()
    el = (time.perf_counter() - t0) / 1000 * 1e6
    s.synchronize()
    print(f"{name:34s} {el:7.2f} us/call (host)")
t.close()
