import sys, os
sys.path.insert(0, "/root/repo")
import torch, numpy as np
import synth, paper_2310_05205_b200 as G
cfg = synth.CONFIGS["c1"]
dt = {"u8": G.GEAR_U8, "i32": G.GEAR_I32, "f32": G.GEAR_F32}
for R, mb in ((1, 4096), (4, 4096), (1, 64)):
    t = G.Table(1024, cfg.seq_len, [G.Column(c.name, dt[c.dtype], c.shape) for c in cfg.cols], None, shards_per_rank=R, max_batch=mb)
    rows = [torch.zeros((1024 // R, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
    for s in range(R):
        G.gear_insert(t.handle, s, 1024 // R, rows, synth.priorities(1024 // R), None, None)
    idx = torch.empty(64, dtype=torch.int64, device="cuda"); w = torch.empty(64, dtype=torch.float32, device="cuda")
    try:
        G.gear_sample(t.handle, G.GEAR_PRIORITIZED | G.GEAR_SAMPLE_OWNER_AFFINE, 64, 5, 0.4, idx, w)
        torch.cuda.synchronize(); print("R", R, "mb", mb, "ok", idx[:4].tolist())
    except Exception as e:
        print("R", R, "mb", mb, "FAIL", e); break
    t.close()
