"""Multi-process (gloo, CPU) tests of the N>1 host logic.

* the NCCL unique id of the C-ABI is broadcast through torch.distributed
  exactly as the binding does (comm_from_torch_distributed's first half);
* the sharded selection protocol the GPU path implements -- each rank scans
  only its shard, all-gathers the 16-byte shard totals, and resolves its own
  slice of the global draw against the owner's CDF -- reproduces the
  unsharded oracle (shard-count invariance);
* the decentralised FIFO/LIFO protocol: local top-K per
  shard, all-gather of candidates, identical merge on every rank, equals the
  oracle's global order;
* bench.py's max-over-ranks reduction of step times.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    port = _port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    ps = [ctx.Process(target=_entry, args=(fn, r, world, port, q, args)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = [q.get() for _ in range(world)]
    for r in res:
        assert r == "ok", r


def _entry(fn, rank, world, port, q, args):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        globals()[fn](rank, world, *args)
        dist.destroy_process_group()
        q.put("ok")
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")


# ---------------------------------------------------------------- workers
def _w_unique_id(rank, world):
    import paper_2310_05205_b200 as gear
    obj = [gear.gear_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    got = [None] * world
    dist.all_gather_object(got, obj[0])
    assert len(obj[0]) == 128 and all(g == got[0] for g in got)


def _w_sharded_sampling(rank, world, shards_per_rank, strategy):
    import oracle
    R = shards_per_rank
    S = world * R
    Cs = 257                                   # odd: misaligned shard starts
    rng = np.random.default_rng(42)
    key = rng.integers(0, 1 << 20, size=S * Cs).astype(np.uint64)
    key[rng.random(S * Cs) < 0.2] = 0
    if strategy == oracle.UNIFORM:
        wts = (key > 0).astype(np.uint64)
    else:
        wts = key
    B, seed = 96, 0xABCDEF
    # local: this rank's R shards -> CDFs and totals
    mine = range(rank * R, (rank + 1) * R)
    cdfs = {s: oracle.cdf(wts[s * Cs:(s + 1) * Cs]) for s in mine}
    tot = torch.tensor([int(cdfs[s][-1]) for s in mine], dtype=torch.int64)
    allt = [torch.zeros(R, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allt, tot)                          # the 16-byte totals exchange
    T_s = torch.cat(allt).numpy().astype(np.uint64)
    G = np.cumsum(T_s, dtype=np.uint64)
    T = int(G[-1])
    # owners resolve draws against their CDF: gather every shard's CDF so this
    # rank can search the owner's (the GPU reads it over NVLink instead)
    mats = [None] * world
    dist.all_gather_object(mats, {s: cdfs[s] for s in mine})
    allc = {s: c for m in mats for s, c in m.items()}
    got = []
    for b in range(B):
        j = rank * B + b
        u = oracle.draw(seed, j, T)
        s = int(np.argmax(G > np.uint64(u)))
        excl = int(G[s]) - int(T_s[s])
        i, _ = oracle.inverse(allc[s], u - excl)
        got.append(s * Cs + i)
    st, want, _, _ = oracle.sample(strategy, key, None, Cs, S, world, rank, B, seed, 0.4)
    assert st == 0
    assert np.array_equal(np.array(got, np.uint64), want)


def _w_fifo_merge(rank, world, lifo):
    import oracle
    R, Cs, B = 2, 64, 12
    S = world * R
    K = world * B
    t = oracle.Table(Cs, S, removal=0)
    rng = np.random.default_rng(3)
    for _ in range(S * Cs * 2):                         # wrap every ring
        t.insert(int(rng.integers(0, S)), [1.0])
    t.key[rng.random(S * Cs) < 0.3] = 0
    # local candidates: the K oldest (newest) selectable of each own shard
    cands = []
    for s in range(rank * R, (rank + 1) * R):
        g = np.arange(s * Cs, (s + 1) * Cs)
        g = g[t.key[g] > 0]
        order = np.argsort(t.seq[g], kind="stable")
        g = g[order][::-1] if lifo else g[order]
        cands += [(int(t.seq[x]), s, int(x)) for x in g[:K]]
    allc = [None] * world
    dist.all_gather_object(allc, cands)                 # O(m k) exchange
    merged = sorted((c for cs in allc for c in cs), reverse=bool(lifo))
    mine = [g for _, _, g in merged[rank * B:(rank + 1) * B]]
    st, want, _, _ = t.sample(oracle.LIFO if lifo else oracle.FIFO, world, rank, B, 0)
    assert st == 0 and mine == [int(x) for x in want]


def _w_topk_merge(rank, world):
    """Decentralised TopK: each rank's shards offer their
    local top-K by (key desc, id asc); the merge of the all-gathered lists
    equals the oracle's global TopK."""
    import oracle
    R, Cs, B = 2, 80, 9
    S, K = world * R, world * B
    rng = np.random.default_rng(8)
    key = rng.integers(0, 5, size=S * Cs).astype(np.uint64)     # heavy ties
    cands = []
    for s in range(rank * R, (rank + 1) * R):
        g = np.arange(s * Cs, (s + 1) * Cs)
        g = g[key[g] > 0]
        top = sorted(g.tolist(), key=lambda x: (-int(key[x]), x))[:K]
        cands += [(-int(key[x]), x) for x in top]
    allc = [None] * world
    dist.all_gather_object(allc, cands)
    merged = sorted(c for cs in allc for c in cs)
    mine = [g for _, g in merged[rank * B:(rank + 1) * B]]
    st, want, _, _ = oracle.sample(oracle.TOPK, key, None, Cs, S, world, rank, B, 0)
    assert st == 0 and mine == [int(x) for x in want]


def _w_max_over_ranks(rank, world):
    ms = torch.tensor([1.0 + rank, 10.0 - rank])
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    assert ms.tolist() == [float(world), 10.0]


def _w_sampling_all(rank, world):
    for R in ((1, 2) if world == 2 else (1,)):
        for strategy in (2, 4):                        # UNIFORM, PRIORITIZED
            _w_sharded_sampling(rank, world, R, strategy)


def _w_misc(rank, world):
    _w_unique_id(rank, world)
    _w_max_over_ranks(rank, world)
    for lifo in (0, 1):
        _w_fifo_merge(rank, world, lifo)
    _w_topk_merge(rank, world)


# ---------------------------------------------------------------- tests
def test_unique_id_fifo_merge_and_max_gloo():
    _run("_w_misc", 2)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_sampling_equals_oracle(world):
    _run("_w_sampling_all", world)
