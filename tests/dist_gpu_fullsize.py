"""Full-size multi-rank parity (launched by tests/test_gpu_multi.py through
torchrun): BASELINE.json configs[1] (c2: 100,000 x 847,080 B, 84.7 GB of HBM)
sharded over W ranks exactly as bench.py builds it, then prioritized steps
with collective updates under both assignments of the global batch (DESIGN.md
Q19 owner-affine, Q9 contiguous).  Every rank checks its sampled ids and IS
weights against the unsharded oracle and EVERY collected row of its slice --
rows of peer shards read through CUDA-IPC mappings -- against the rows of the
oracle's ids regenerated on the GPU (synth.fill_rows_ids).

With GEAR_SHARED_DEVICE=1 the W rank processes share one GPU (gloo bootstrap,
gear_comm_create_host): the 84.7 GB table fits one B200, so the driver's
1-GPU box runs the W=2 full-size path.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402


def main():
    W = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    if os.environ.get("GEAR_SHARED_DEVICE", "0") == "1":
        local = 0
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        comm = gear.comm_from_process_group(0)
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = gear.comm_from_torch_distributed(local)
    cfg = synth.CONFIGS["c2"]
    capacity, _ = bench.scaled_capacity(cfg, W)
    Cs = capacity // W
    stream = torch.cuda.Stream()
    t, prio_all = bench.build_table(cfg, comm, W, rank, capacity, stream)
    o = oracle.Table(Cs, W)
    for s in range(W):
        st, _ = o.insert(s, prio_all[s * Cs:(s + 1) * Cs])
        assert st == 0
    dist.barrier()
    key, _, _ = t.read_state()
    assert np.array_equal(key, o.key[rank * Cs:(rank + 1) * Cs]), "keys after the build"
    B = cfg.batch
    idx = torch.empty(B, dtype=torch.int64, device="cuda")
    w = torch.empty(B, dtype=torch.float32, device="cuda")
    outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
    want = [torch.empty_like(x) for x in outs]
    plan = [True, True, False, True, False]        # owner-affine / contiguous per step
    for step, affine in enumerate(plan):
        seed = synth.SAMPLE_SEED_BASE + 50 + step
        flags = gear.GEAR_SAMPLE_OWNER_AFFINE if affine else 0
        gear.gear_sample(t.handle, gear.GEAR_PRIORITIZED, B, seed, cfg.beta, idx, w, None, None,
                         stream, flags=flags)
        gear.gear_collect(t.handle, B, idx, list(range(len(outs))), outs, stream)
        p = synth.priorities(B, seed=2000 + 10 * step + rank)
        gear.gear_update_priorities(t.handle, B, idx, torch.from_numpy(p).cuda(), gear.GEAR_F64,
                                    None, stream)
        stream.synchronize()
        st, oi, ow, _ = o.sample(oracle.PRIORITIZED, W, rank, B, seed, cfg.beta, owner_affine=affine)
        assert st == 0
        gi = idx.cpu().numpy().view(np.uint64)
        assert np.array_equal(gi, oi), f"step {step} (affine={affine}): ids differ"
        np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-6, atol=0)
        d_ids = torch.from_numpy(oi.view(np.int64)).cuda()
        for c, rb in enumerate(t.row_bytes):
            synth.fill_rows_ids(want[c].data_ptr(), d_ids.data_ptr(), B, rb, c,
                                stream=stream.cuda_stream)
        stream.synchronize()
        for c in range(len(outs)):
            if not torch.equal(outs[c], want[c]):
                bad = (outs[c] != want[c]).any(dim=1).nonzero().flatten()[:8].tolist()
                raise AssertionError(f"step {step} (affine={affine}) column {c}: rows {bad} differ")
        remote = float(np.mean((gi // np.uint64(Cs)) != rank))
        lists = [None] * W
        dist.all_gather_object(lists, (gi, p))
        for r in range(W):                        # (rank, position) order, last writer wins
            o.update(lists[r][0], lists[r][1])
        if rank == 0:
            print(f"step {step} affine={affine}: {B} ids, weights and every row of "
                  f"{sum(t.row_bytes)} B ok (remote rows {remote:.3f})", flush=True)
    key, _, _ = t.read_state()
    assert np.array_equal(key, o.key[rank * Cs:(rank + 1) * Cs]), "keys after the collective updates"
    err, _ = t.sync()
    assert err == 0, err
    t.close()
    gear.gear_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank}: full-size multi-rank parity ok (W={W}, N={capacity})", flush=True)


if __name__ == "__main__":
    main()
