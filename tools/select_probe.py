"""Selection cost per strategy at W ranks (development probe): gear_sample alone,
30 back-to-back calls after 5 warm-ups on the c2 table, CUDA events, max over
ranks; owner-affine as in bench.py.  Run under torchrun for W > 1."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
comm = None
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = gear.comm_from_torch_distributed(local)
cfg = synth.CONFIGS["c2"]
s = torch.cuda.Stream()
t, _ = bench.build_table(cfg, comm, world, rank, cfg.capacity, s)
B = cfg.batch
idx = torch.empty(B, dtype=torch.int64, device="cuda")
w = torch.empty(B, dtype=torch.float32, device="cuda")
res = {}
for name in ("prioritized", "fifo", "topk"):
    strat = gear.STRATEGIES[name] | (gear.GEAR_SAMPLE_OWNER_AFFINE if world > 1 else 0)
    for i in range(5):
        gear.gear_sample(t.handle, strat, B, i, 0.4, idx, w, None, None, s)
    s.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(30):
        gear.gear_sample(t.handle, strat, B, 100 + i, 0.4, idx, w, None, None, s)
    e1.record(s)
    s.synchronize()
    us = torch.tensor([e0.elapsed_time(e1) / 30 * 1e3], device="cuda")
    if world > 1:
        dist.all_reduce(us, op=dist.ReduceOp.MAX)
    res[name] = round(float(us.item()), 2)
assert t.sync()[0] == 0
if rank == 0:
    print(json.dumps({"W": world, "B": B, "us_per_sample": res}), flush=True)
t.close()
if world > 1:
    dist.destroy_process_group()
