"""Multi-GPU parity (one process per GPU, NCCL over NVLink): launched by
tests/test_gpu_multi.py as

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/dist_gpu_parity.py

Every rank runs the SPMD hot path on its shard(s) of a table sharded by
trajectory id, and checks its slice against the unsharded CPU oracle:
sampled ids (bit-exact), IS weights (1e-6 rel), collected rows -- including
rows of peer shards read over NVLink (DEVICE columns) and rows of other
ranks' host shards read zero-copy over this GPU's PCIe (HOST columns) -- and
the keys after collective priority updates.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

OS = {gear.GEAR_FIFO: oracle.FIFO, gear.GEAR_LIFO: oracle.LIFO, gear.GEAR_UNIFORM: oracle.UNIFORM,
      gear.GEAR_WEIGHTED: oracle.WEIGHTED, gear.GEAR_PRIORITIZED: oracle.PRIORITIZED,
      gear.GEAR_TOPK: oracle.TOPK}


def write_rows_in_place(t, c, placement, local, rows, nrows, rb):
    """Rows of rank-local slots `local` of column c, written at gear_column_base."""
    import ctypes
    base = t.column_base(c)
    if placement == gear.GEAR_DEVICE:
        class _View:
            __cuda_array_interface__ = {"shape": (nrows, rb), "typestr": "|u1",
                                        "data": (base, False), "version": 3}
        col = torch.as_tensor(_View(), device="cuda")
        col[torch.from_numpy(local).cuda()] = torch.from_numpy(rows).cuda()
    else:
        col = np.ctypeslib.as_array(ctypes.cast(base, ctypes.POINTER(ctypes.c_uint8)),
                                    shape=(nrows, rb))
        col[local] = rows
    torch.cuda.synchronize()


def run_case(comm, W, rank, R, placements, removal, Cs=700, B=40, steps=3, xchg=1):
    dt = [gear.GEAR_F32, gear.GEAR_U8, gear.GEAR_I32]
    shapes = [(5,), (3,), ()]
    cols = [gear.Column(f"c{i}", dt[i % 3], shapes[i % 3], p) for i, p in enumerate(placements)]
    S = W * R
    N = S * Cs
    t = gear.Table(N, 4, cols, comm, shards_per_rank=R, removal=removal, max_batch=1024)
    gear.gear_table_set_tuning(t.handle, "peer_xchg", xchg)
    o = oracle.Table(Cs, S, removal=removal)
    rb = t.row_bytes
    content = np.full(N, -1, np.int64)
    prio_all = synth.priorities(2 * N, seed=9, zero_frac=0.1)
    rng = np.random.default_rng(5)
    plan = []                                   # (shard, n) inserts, same on every rank
    for s in range(S):
        k = 0
        while k < int(Cs * 1.25):
            b = int(rng.integers(1, 400))
            b = min(b, int(Cs * 1.25) - k)
            plan.append((s, k, b))
            k += b
    for s, k, b in plan:
        traj = np.arange(s * 2 * Cs + k, s * 2 * Cs + k + b)
        p = prio_all[s * 2 * Cs + k: s * 2 * Cs + k + b]
        st, oidx = o.insert(s, p)
        content[oidx.astype(np.int64)] = traj
        if s // R == rank:
            rows = [torch.from_numpy(synth.row_bytes_of(c, traj, rb[c])).cuda() for c in range(len(cols))]
            out = np.zeros(b, np.uint64)
            t.insert(s, rows, p, out)
            assert np.array_equal(out, oidx), "insert slots differ"
    torch.cuda.synchronize()
    dist.barrier()
    key, seq, gen = t.read_state()
    lo, hi = rank * R * Cs, (rank + 1) * R * Cs
    assert np.array_equal(key, o.key[lo:hi]) and np.array_equal(seq, o.seq[lo:hi])
    assert np.array_equal(gen, o.gen[lo:hi])

    # split writer API (reading Q21): every rank allocates in its own shards,
    # writes the rows in place at gear_column_base, then commits
    for s in range(S):
        n = 30
        st, oids = o.allocate(s, n)
        assert st == 0
        traj = np.arange(10 ** 7 + 1000 * s, 10 ** 7 + 1000 * s + n)
        content[oids.astype(np.int64)] = traj
        pc = synth.priorities(n, seed=77 + s)
        assert o.commit(s, oids, pc) == 0
        if s // R != rank:
            continue
        ids = torch.empty(n, dtype=torch.int64, device="cuda")
        t.allocate(s, n, ids)
        torch.cuda.synchronize()
        gids = ids.cpu().numpy().view(np.uint64)
        assert np.array_equal(gids, oids), "allocated slots differ"
        local = (gids - np.uint64(lo)).astype(np.int64)
        for c in range(len(cols)):
            rows = synth.row_bytes_of(c, traj, rb[c])
            write_rows_in_place(t, c, placements[c], local, rows, R * Cs, rb[c])
        t.commit(s, ids, torch.from_numpy(pc).cuda())
    torch.cuda.synchronize()
    dist.barrier()
    err, _ = t.sync()
    assert err == 0, err
    key, seq, gen = t.read_state()
    assert np.array_equal(key, o.key[lo:hi]) and np.array_equal(seq, o.seq[lo:hi])
    assert np.array_equal(gen, o.gen[lo:hi])

    for step in range(steps):
        for strat in (gear.GEAR_UNIFORM, gear.GEAR_WEIGHTED, gear.GEAR_PRIORITIZED, gear.GEAR_FIFO,
                      gear.GEAR_LIFO, gear.GEAR_TOPK):
            seed = synth.SAMPLE_SEED_BASE + 100 * step + strat
            idx = torch.empty(B, dtype=torch.int64, device="cuda")
            w = torch.empty(B, dtype=torch.float32, device="cuda")
            pr = torch.empty(B, dtype=torch.float64, device="cuda")
            t.sample(strat, B, seed, 0.4, idx, w, pr)
            torch.cuda.synchronize()
            st, oi, ow, op = o.sample(OS[strat], W, rank, B, seed, 0.4)
            assert st == 0, st
            gi = idx.cpu().numpy().view(np.uint64)
            assert np.array_equal(gi, oi), f"strategy {strat}: ids differ at {np.nonzero(gi != oi)[0][:8]}"
            np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-6)
            assert np.array_equal(pr.cpu().numpy(), op)
            outs = [torch.empty((B, r), dtype=torch.uint8, device="cuda") for r in rb]
            t.collect(idx, list(range(len(cols))), outs)
            torch.cuda.synchronize()
            for c in range(len(cols)):
                want = synth.row_bytes_of(c, content[oi.astype(np.int64)], rb[c])
                assert np.array_equal(outs[c].cpu().numpy(), want), f"collect column {c}"
            err, _ = t.sync()
            assert err == 0, err
            # owner-affine assignment of the same global batch (reading Q19)
            ia = torch.empty(B, dtype=torch.int64, device="cuda")
            wa = torch.empty(B, dtype=torch.float32, device="cuda")
            t.sample(strat | gear.GEAR_SAMPLE_OWNER_AFFINE, B, seed, 0.4, ia, wa)
            torch.cuda.synchronize()
            st, oa, owa, _ = o.sample(OS[strat], W, rank, B, seed, 0.4, owner_affine=True)
            ga = ia.cpu().numpy().view(np.uint64)
            assert st == 0 and np.array_equal(ga, oa), f"strategy {strat}: owner-affine ids differ"
            np.testing.assert_allclose(wa.cpu().numpy(), owa, rtol=1e-6)
            t.collect(ia, list(range(len(cols))), outs)
            torch.cuda.synchronize()
            for c in range(len(cols)):
                want = synth.row_bytes_of(c, content[oa.astype(np.int64)], rb[c])
                assert np.array_equal(outs[c].cpu().numpy(), want), f"affine collect column {c}"
        # collective update: every rank updates its own sampled ids
        newp = np.random.default_rng(1000 * step + rank).lognormal(0, 1, B)
        newp[:3] = 0.0
        gear.gear_update_priorities(t.handle, B, idx, torch.from_numpy(newp).cuda(), gear.GEAR_F64)
        torch.cuda.synchronize()
        lists = [None] * W
        dist.all_gather_object(lists, (gi, newp))
        for r in range(W):                             # (rank, position) order
            o.update(lists[r][0], lists[r][1])
        key, _, _ = t.read_state()
        assert np.array_equal(key, o.key[lo:hi]), "keys after the collective update"
    t.close()


def run_graph_case(comm, W, rank, R=2, Cs=500, B=48, reps=4):
    """Every rank captures sample(owner-affine, device seed) -> collect ->
    update once as a CUDA graph and replays it: the mailbox epochs, the CDF
    parity, the update epoch and the seed are device-resident, so each replay
    is a new collective step and must match the oracle."""
    cols = [gear.Column("a", gear.GEAR_F32, (6,)), gear.Column("b", gear.GEAR_U8, (5,))]
    S = W * R
    N = S * Cs
    t = gear.Table(N, 2, cols, comm, shards_per_rank=R, max_batch=256)
    o = oracle.Table(Cs, S)
    prio_all = synth.priorities(N, seed=21, zero_frac=0.05)
    for s in range(S):
        st, oidx = o.insert(s, prio_all[s * Cs:(s + 1) * Cs])
        if s // R == rank:
            traj = np.arange(s * Cs, (s + 1) * Cs)
            rows = [torch.from_numpy(synth.row_bytes_of(c, traj, t.row_bytes[c])).cuda() for c in range(2)]
            t.insert(s, rows, prio_all[s * Cs:(s + 1) * Cs])
    torch.cuda.synchronize()
    dist.barrier()
    seed0 = 777
    gear.gear_table_set_tuning(t.handle, "device_seed", seed0)
    idx = torch.empty(B, dtype=torch.int64, device="cuda")
    w = torch.empty(B, dtype=torch.float32, device="cuda")
    outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
    newp = [np.random.default_rng(50 + r).lognormal(0, 1, B) for r in range(W)]
    dnewp = torch.from_numpy(newp[rank]).cuda()
    strat = gear.GEAR_PRIORITIZED | gear.GEAR_SAMPLE_OWNER_AFFINE | gear.GEAR_SAMPLE_DEVICE_SEED

    def step():
        gear.gear_sample(t.handle, strat, B, 0, 0.4, idx, w)
        gear.gear_collect(t.handle, B, idx, [0, 1], outs)
        gear.gear_update_priorities(t.handle, B, idx, dnewp, gear.GEAR_F64)

    step()                                   # eager step (seed0), also warms up
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    sgraph = torch.cuda.Stream()
    sgraph.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(sgraph):
        with torch.cuda.graph(g, stream=sgraph, capture_error_mode="thread_local"):
            step()
    torch.cuda.synchronize()
    dist.barrier()
    got = []
    with torch.cuda.stream(sgraph):
        for _ in range(reps):
            g.replay()
            sgraph.synchronize()
            got.append((idx.cpu().numpy().view(np.uint64).copy(), w.cpu().numpy().copy(),
                        [x.cpu().numpy().copy() for x in outs]))
    err, _ = t.sync()
    assert err == 0, err
    content = np.arange(N)
    for i in range(reps + 1):
        seed = seed0 + i
        lists = []
        for r in range(W):
            st, oi, ow, _ = o.sample(oracle.PRIORITIZED, W, r, B, seed, 0.4, owner_affine=True)
            assert st == 0
            lists.append(oi)
            if r == rank and i >= 1:
                gi, gw, gouts = got[i - 1]
                assert np.array_equal(gi, oi), f"graph replay {i}: ids differ"
                np.testing.assert_allclose(gw, ow, rtol=1e-6)
                for c in range(2):
                    want = synth.row_bytes_of(c, content[oi.astype(np.int64)], t.row_bytes[c])
                    assert np.array_equal(gouts[c], want)
        for r in range(W):
            o.update(lists[r], newp[r])
    key, _, _ = t.read_state()
    lo, hi = rank * R * Cs, (rank + 1) * R * Cs
    assert np.array_equal(key, o.key[lo:hi]), "keys after the replayed collective updates"
    t.close()


def run_fuzz_case(comm, W, rank, R=2, Cs=400, steps=150, seed=11):
    """Random collective operation sequences (inserts, allocate / commit,
    updates, samples of every strategy plain and owner-affine, collects), the
    same sequence on every rank, each result compared with the oracle --
    exercises the mailbox epochs across arbitrary interleavings."""
    cols = [gear.Column("a", gear.GEAR_F32, (3,), gear.GEAR_DEVICE),
            gear.Column("b", gear.GEAR_U8, (5,), gear.GEAR_HOST)]
    S = W * R
    N = S * Cs
    t = gear.Table(N, 2, cols, comm, shards_per_rank=R, max_batch=256)
    o = oracle.Table(Cs, S)
    rb = t.row_bytes
    content = np.full(N, -1, np.int64)
    rng = np.random.default_rng(seed)            # identical on every rank
    lo, hi = rank * R * Cs, (rank + 1) * R * Cs
    next_traj = 0
    strategies = [gear.GEAR_UNIFORM, gear.GEAR_WEIGHTED, gear.GEAR_PRIORITIZED, gear.GEAR_FIFO,
                  gear.GEAR_LIFO, gear.GEAR_TOPK]
    for step in range(steps):
        op = int(rng.integers(0, 5))
        if op == 0:                              # every shard gets an insert
            for s in range(S):
                n = int(rng.integers(1, 150))
                p = synth.priorities(n, seed=1000 * step + s, zero_frac=0.1)
                traj = np.arange(next_traj, next_traj + n)
                next_traj += n
                st, oidx = o.insert(s, p)
                content[oidx.astype(np.int64)] = traj
                if s // R == rank:
                    rows = [torch.from_numpy(synth.row_bytes_of(c, traj, rb[c])).cuda()
                            for c in range(len(cols))]
                    out = np.zeros(n, np.uint64)
                    t.insert(s, rows, p, out)
                    assert np.array_equal(out, oidx), "insert slots differ"
        elif op == 1:                            # allocate -> rows in place -> commit
            for s in range(S):
                n = int(rng.integers(1, 20))
                st, oids = o.allocate(s, n)
                if st != 0:
                    continue
                traj = np.arange(next_traj, next_traj + n)
                next_traj += n
                content[oids.astype(np.int64)] = traj
                pc = synth.priorities(n, seed=7 * step + s)
                o.commit(s, oids, pc)
                if s // R == rank:
                    ids = torch.empty(n, dtype=torch.int64, device="cuda")
                    t.allocate(s, n, ids)
                    torch.cuda.synchronize()
                    assert np.array_equal(ids.cpu().numpy().view(np.uint64), oids)
                    local = (oids - np.uint64(lo)).astype(np.int64)
                    for c in range(len(cols)):
                        write_rows_in_place(t, c, cols[c].placement, local,
                                            synth.row_bytes_of(c, traj, rb[c]), R * Cs, rb[c])
                    t.commit(s, ids, torch.from_numpy(pc).cuda())
        elif op == 2:                            # collective update of random ids
            n = int(rng.integers(1, 200))
            lists = [(rng.integers(0, N, n).astype(np.uint64), rng.lognormal(0, 1, n))
                     for _ in range(W)]
            ids, p = lists[rank]
            gear.gear_update_priorities(t.handle, n, torch.from_numpy(ids.view(np.int64)).cuda(),
                                        torch.from_numpy(p).cuda(), gear.GEAR_F64)
            for r in range(W):
                o.update(lists[r][0], lists[r][1])
            torch.cuda.synchronize()
            err, _ = t.sync()                    # never-inserted / ongoing ids: stale
            assert err & ~gear.GEAR_DEVERR_STALE == 0, err
        else:                                    # sample (+ collect)
            strat = strategies[int(rng.integers(0, len(strategies)))]
            affine = bool(rng.integers(0, 2))
            B = int(rng.integers(1, 100))
            sd = int(rng.integers(0, 1 << 30))
            idx = torch.empty(B, dtype=torch.int64, device="cuda")
            w = torch.empty(B, dtype=torch.float32, device="cuda")
            t.sample(strat | (gear.GEAR_SAMPLE_OWNER_AFFINE if affine else 0), B, sd, 0.4, idx, w)
            torch.cuda.synchronize()
            st, oi, ow, _ = o.sample(OS[strat], W, rank, B, sd, 0.4, owner_affine=affine)
            gi = idx.cpu().numpy().view(np.uint64)
            err, _ = t.sync()
            if st == oracle.EMPTY:
                assert err & gear.GEAR_DEVERR_EMPTY
                continue
            assert st == 0 and err == 0, (st, err)
            assert np.array_equal(gi, oi), f"step {step} strategy {strat}: ids differ"
            np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-6)
            outs = [torch.empty((B, r), dtype=torch.uint8, device="cuda") for r in rb]
            t.collect(idx, list(range(len(cols))), outs)
            torch.cuda.synchronize()
            for c in range(len(cols)):
                want = synth.row_bytes_of(c, content[oi.astype(np.int64)], rb[c])
                assert np.array_equal(outs[c].cpu().numpy(), want), f"step {step} column {c}"
        torch.cuda.synchronize()
        dist.barrier()
        key, sq, gen = t.read_state()
        assert np.array_equal(key, o.key[lo:hi]) and np.array_equal(sq, o.seq[lo:hi])
        assert np.array_equal(gen, o.gen[lo:hi])
    t.close()


def run_host_comm_capture_case(comm, W, rank):
    """With a host-bootstrapped comm the peer_xchg = 0 exchanges go through the
    host all-gather: refused (UNSUPPORTED) inside CUDA-graph capture, on every
    rank alike, and the table still works afterwards."""
    cols = [gear.Column("a", gear.GEAR_U8, (4,))]
    t = gear.Table(W * 64, 1, cols, comm, max_batch=64)
    t.insert(rank, [torch.zeros((64, 4), dtype=torch.uint8, device="cuda")], np.ones(64))
    torch.cuda.synchronize()
    dist.barrier()
    gear.gear_table_set_tuning(t.handle, "peer_xchg", 0)
    idx = torch.empty(16, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    refused = False
    try:
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
                gear.gear_sample(t.handle, gear.GEAR_UNIFORM, 16, 3, 0.0, idx)
    except gear.GearError as e:
        refused = e.status == gear.GEAR_ERR_UNSUPPORTED
    except RuntimeError:      # the capture itself was invalidated after the refusal
        refused = True
    assert refused, "an all-gather through the host callback was captured"
    torch.cuda.synchronize()
    dist.barrier()
    gear.gear_sample(t.handle, gear.GEAR_UNIFORM, 16, 3, 0.0, idx)   # eager: fine
    torch.cuda.synchronize()
    assert np.all(idx.cpu().numpy() < W * 64)
    dist.barrier()
    t.close()


def run_topk_large_case(comm, W, rank, Cs=20000, B=4096):
    """TopK with K = W*B >= 8192 candidates: the sorted-runs + merge-rank sort
    (topk.cu) feeding every peer's mailbox, against the oracle (Q20)."""
    cols = [gear.Column("x", gear.GEAR_U8, (4,))]
    N = W * Cs
    t = gear.Table(N, 1, cols, comm, max_batch=B)
    o = oracle.Table(Cs, W)
    rng = np.random.default_rng(123)
    vals = np.array([0.0, 0.5, 1.0, 2.0, 3.0])
    prio = np.where(rng.random(N) < 0.5, vals[rng.integers(0, len(vals), N)],
                    synth.priorities(N, seed=3, zero_frac=0.0))
    for s in range(W):
        p = prio[s * Cs:(s + 1) * Cs]
        st, oidx = o.insert(s, p)
        if s == rank:
            out = np.zeros(Cs, np.uint64)
            t.insert(s, [torch.zeros((Cs, 4), dtype=torch.uint8, device="cuda")], p, out)
            assert np.array_equal(out, oidx)
    torch.cuda.synchronize()
    dist.barrier()
    for b in (B, B // 2 + 3):
        idx = torch.empty(b, dtype=torch.int64, device="cuda")
        t.sample(gear.GEAR_TOPK, b, 0, 0.4, idx)
        torch.cuda.synchronize()
        st, oi, _, _ = o.sample(oracle.TOPK, W, rank, b, 0, 0.4)
        assert st == 0, st
        gi = idx.cpu().numpy().view(np.uint64)
        assert np.array_equal(gi, oi), f"TopK K={W * b}: ids differ at {np.nonzero(gi != oi)[0][:8]}"
    err, _ = t.sync()
    assert err == 0, err
    t.close()


def run_timeout_case(comm, W, rank, R=1, Cs=256, B=32):
    """A broken SPMD sequence: only rank 0 calls gear_sample and then
    gear_update_priorities.  Its mailbox waits time out after ~4 s; the
    sample must return GEAR_IDX_NONE everywhere (not ids drawn from stale
    totals) and latch TIMEOUT, and the update must change no key."""
    cols = [gear.Column("a", gear.GEAR_U8, (8,))]
    t = gear.Table(W * R * Cs, 1, cols, comm, shards_per_rank=R, max_batch=256)
    for ls in range(R):
        s = rank * R + ls
        t.insert(s, [torch.zeros((Cs, 8), dtype=torch.uint8, device="cuda")],
                 synth.priorities(Cs, seed=s) + 0.5)
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        key0, _, _ = t.read_state()
        idx = torch.zeros(B, dtype=torch.int64, device="cuda")
        w = torch.empty(B, dtype=torch.float32, device="cuda")
        t.sample(gear.GEAR_PRIORITIZED, B, 5, 0.4, idx, w)
        torch.cuda.synchronize()
        err, _ = t.sync()
        assert err & gear.GEAR_DEVERR_TIMEOUT and not err & gear.GEAR_DEVERR_EMPTY, err
        assert np.all(idx.cpu().numpy().view(np.uint64) == np.uint64(gear.GEAR_IDX_NONE))
        ids = torch.arange(B, dtype=torch.int64, device="cuda")
        gear.gear_update_priorities(t.handle, B, ids, torch.full((B,), 7.0, dtype=torch.float64,
                                                                device="cuda"), gear.GEAR_F64)
        torch.cuda.synchronize()
        err, _ = t.sync()
        assert err & gear.GEAR_DEVERR_TIMEOUT, err
        key1, _, _ = t.read_state()
        assert np.array_equal(key0, key1), "a timed-out update changed keys"
    dist.barrier()
    t.close()


def main():
    W = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    shared = os.environ.get("GEAR_SHARED_DEVICE", "0") == "1"
    if shared:
        # every rank on cuda:0, bootstrapped through gloo (NCCL refuses two
        # ranks on one device): the same mailbox / IPC / shared-shm device path
        local = 0
        torch.cuda.set_device(0)
        dist.init_process_group("gloo")
        comm = gear.comm_from_process_group(0)
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = gear.comm_from_torch_distributed(local)
    D, H = gear.GEAR_DEVICE, gear.GEAR_HOST
    quick = os.environ.get("GEAR_DIST_QUICK", "0") == "1"   # smoke(): one case + graph replay
    cases = [(1, [D, D, D], 0, 1), (2, [D, D, D], 1, 1), (1, [H, H, H], 0, 1),
             (2, [D, H, D], 0, 1), (1, [D, D, D], 0, 0), (2, [D, H, D], 1, 0)]
    if quick:
        cases = [(2, [D, H, D], 0, 1)]
    for R, pl, removal, xchg in cases:
        run_case(comm, W, rank, R, pl, removal, xchg=xchg, steps=1 if quick else 3)
        dist.barrier()
        if rank == 0:
            print(f"case R={R} placements={pl} removal={removal} peer_xchg={xchg}: ok", flush=True)
    run_graph_case(comm, W, rank, reps=4 if quick else 48)
    dist.barrier()
    if rank == 0:
        print("case graph replay (owner-affine, device seed): ok", flush=True)
    if not quick:
        # GEAR_FUZZ_STEPS / GEAR_FUZZ_SEEDS: longer soak runs of the same case
        fuzz_steps = int(os.environ.get("GEAR_FUZZ_STEPS", "150"))
        for fseed in [int(x) for x in os.environ.get("GEAR_FUZZ_SEEDS", "11").split(",")]:
            run_fuzz_case(comm, W, rank, steps=fuzz_steps, seed=fseed)
            dist.barrier()
            if rank == 0:
                print(f"case random collective sequences (seed {fseed}, {fuzz_steps} steps): ok",
                      flush=True)
        if shared:
            run_host_comm_capture_case(comm, W, rank)
            dist.barrier()
            if rank == 0:
                print("case host comm: all-gather refused inside graph capture: ok", flush=True)
        run_topk_large_case(comm, W, rank)
        dist.barrier()
        if rank == 0:
            print(f"case TopK with K = {W} x 4096 (sorted runs + merge ranks, mailboxes): ok", flush=True)
        run_timeout_case(comm, W, rank)
        dist.barrier()
        if rank == 0:
            print("case broken SPMD sequence (mailbox timeout -> GEAR_IDX_NONE, no key change): ok",
                  flush=True)
    gear.gear_comm_destroy(comm)
    dist.destroy_process_group()
    print(f"rank {rank}: all multi-GPU parity cases ok ({'shared device, host bootstrap' if shared else 'one GPU per rank, NCCL bootstrap'})",
          flush=True)


if __name__ == "__main__":
    main()
