"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Indices, keys, seq/gen and collected bytes bit-exact;
IS weights within 1e-6 relative (north star); q/T probabilities bit-exact
(correctly rounded division on both sides)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2310_05205_b200 as gear
    gear.load()
    return torch


def _pair(**kw):
    from gpu_harness import Pair
    return Pair(**kw)


C1 = synth.CONFIGS["c1"]
G = __import__("paper_2310_05205_b200")


@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("placement", ["device", "host"])
def test_c1_sample_collect_update(torch_cuda, R, placement):
    """c1 shapes: insert every row, then steps of UNIFORM / WEIGHTED /
    PRIORITIZED sampling, collection of the sampled rows and priority
    updates of them (with duplicates), for 1/2/4/8 shards (virtual world:
    the result must not depend on the shard count)."""
    P = _pair(capacity=C1.capacity, seq_len=C1.seq_len, colspecs=C1.cols, R=R, placement=placement)
    P.fill(synth.priorities(C1.capacity, seed=1, zero_frac=0.10))
    P.check_state()
    rng = np.random.default_rng(7)
    for step in range(6):
        for strat in (G.GEAR_UNIFORM, G.GEAR_WEIGHTED, G.GEAR_PRIORITIZED):
            idx = P.check_sample(strat, 64, synth.SAMPLE_SEED_BASE + 10 * step + strat, beta=0.4)
            P.check_collect(idx)
        newp = rng.lognormal(0, 1, size=64)
        newp[rng.random(64) < 0.05] = 0.0
        ost, _, err, _ = P.update(idx, newp)
        assert ost == 0 and err == 0
        P.check_state()
    P.close()


def test_scan_multi_tile_ragged(torch_cuda):
    """Shards spanning several 4096-key scan tiles with an odd shard capacity
    (misaligned shard starts, ragged last tile) and a long look-back."""
    cols = [synth.ColSpec("x", "u8", (3,))]
    N = 5 * 20011
    P = _pair(capacity=N, seq_len=1, colspecs=cols, R=5, mirror=True)
    P.fill(synth.priorities(N, seed=3, zero_frac=0.2, sigma=2.0))
    for s in range(4):
        for strat in (G.GEAR_UNIFORM, G.GEAR_PRIORITIZED):
            idx = P.check_sample(strat, 1000, 99 + s, beta=0.6)
    P.check_collect(idx)
    P.close()


def test_single_shard_many_tiles(torch_cuda):
    cols = [synth.ColSpec("x", "i32", (5,))]
    N = 4096 * 37 + 1
    P = _pair(capacity=N, seq_len=2, colspecs=cols, R=1)
    P.fill(synth.priorities(N, seed=4, zero_frac=0.01))
    for s in range(3):
        P.check_sample(G.GEAR_WEIGHTED, 2048, 1234 + s)
    P.close()


def test_zero_weight_and_empty(torch_cuda):
    cols = [synth.ColSpec("x", "f32", ())]
    P = _pair(capacity=3, seq_len=1, colspecs=cols, R=1)
    P.insert(0, [0.0, 5.0, 0.0])
    for strat in (G.GEAR_UNIFORM, G.GEAR_WEIGHTED, G.GEAR_PRIORITIZED):
        idx = P.check_sample(strat, 100, 5)
        assert np.all(idx == 1)
    P.update([1], [0.0])
    for strat in (G.GEAR_UNIFORM, G.GEAR_WEIGHTED, G.GEAR_PRIORITIZED, G.GEAR_FIFO, G.GEAR_LIFO):
        assert P.check_sample(strat, 4, 6) is None    # EMPTY latched, ids = IDX_NONE
    P.close()


@pytest.mark.parametrize("fused", [0, 1])
def test_update_errors_duplicates_and_generations(torch_cuda, fused):
    """Both update paths: the single-CTA fused launch and the two grid-wide
    tag/apply launches."""
    cols = [synth.ColSpec("x", "u8", (8,))]
    P = _pair(capacity=256, seq_len=1, colspecs=cols, R=2)
    G.gear_table_set_tuning(P.t.handle, "update_fused", fused)
    P.insert(0, np.ones(100))
    P.insert(1, np.ones(128))
    rng = np.random.default_rng(11)
    idx = rng.integers(0, 256, size=600).astype(np.uint64)   # includes never-inserted slots
    p = rng.lognormal(0, 2, size=600)
    p[5], p[6], p[7] = np.nan, -1.0, np.inf
    idx[8] = 256                                            # out of range
    idx[9] = np.uint64(G.GEAR_IDX_NONE)                     # padding entry
    ost, ons, err, ns = P.update(idx, p)
    assert bool(ost & 1) == bool(err & G.GEAR_DEVERR_BAD_PRIORITY)
    assert bool(ost & 2) == bool(err & G.GEAR_DEVERR_INDEX_RANGE)
    assert bool(ost & 4) == bool(err & G.GEAR_DEVERR_STALE)
    assert ns == ons and ns > 0
    P.check_state()
    # generation-checked update: half the entries carry a stale generation
    key, seq, gen = P.t.read_state()
    ids = np.arange(0, 100, dtype=np.uint64)
    g = gen[:100].copy()
    g[::2] += 1
    ost, ons, err, ns = P.update(ids, np.full(100, 3.25), gen=g)
    assert ns == ons == 50
    P.check_state()
    # f32 priorities widen exactly
    ost, ons, err, ns = P.update(ids, rng.lognormal(0, 1, 100).astype(np.float32), f32=True)
    P.check_state()
    P.close()


def test_quantize_edges_on_gpu(torch_cuda):
    """Q_F special cases (ties to even, clamps, saturation) against the oracle."""
    cols = [synth.ColSpec("x", "u8", ())]
    P = _pair(capacity=1024, seq_len=1, colspecs=cols, R=1)
    P.insert(0, np.ones(1024))
    vals = [0.0, 2.0 ** -40, 1.0, 1.5, 2.0 ** 30, 1e300, 2.0 ** 20]
    vals += [(k + 0.5) * 2.0 ** -32 for k in range(0, 40)]
    vals += [(6.5 + 2.0 ** -20) * 2.0 ** -32, (7.5 - 2.0 ** -20) * 2.0 ** -32, 5e-324]
    P.update(np.arange(len(vals), dtype=np.uint64), np.array(vals))
    P.check_state()
    P.close()


@pytest.mark.parametrize("levels", [2, 1])
def test_cdf_levels_incremental(torch_cuda, levels):
    """The two-level incremental CDF (default) and the flat look-back CDF give
    the oracle's draws through: a first build, sparse updates (a few dirty
    tiles of a few shards), no-change samples, alternating UNIFORM (indicator)
    and PRIORITIZED (weights) builds -- each CDF buffer remembers its own
    mode -- inserts, and a ragged last tile."""
    cols = [synth.ColSpec("x", "u8", (8,))]
    R, Cs = 3, 10_000                       # 3 tiles per shard, the last ragged
    P = _pair(capacity=Cs * R, seq_len=1, colspecs=cols, R=R)
    G.gear_table_set_tuning(P.t.handle, "cdf_levels", levels)
    rng = np.random.default_rng(5)
    P.fill(synth.priorities(Cs * R, seed=3, zero_frac=0.1))
    seed = 100
    for rnd in range(6):
        strat = G.GEAR_UNIFORM if rnd in (2, 3) else G.GEAR_PRIORITIZED
        P.check_sample(strat, 4096, seed)
        seed += 1
        P.check_sample(strat, 777, seed)    # nothing changed: no rebuild
        seed += 1
        ids = rng.choice(Cs * R, size=int(rng.integers(1, 6)), replace=False).astype(np.uint64)
        P.update(ids, rng.lognormal(0, 3, ids.size) * (rng.random(ids.size) > 0.3))
    P.insert(1, synth.priorities(50, seed=9))
    P.check_sample(G.GEAR_WEIGHTED, 4096, seed)
    P.check_sample(G.GEAR_UNIFORM, 4096, seed + 1)
    G.gear_table_set_tuning(P.t.handle, "cdf_levels", 3 - levels)   # switch layouts
    P.check_sample(G.GEAR_PRIORITIZED, 4096, seed + 2)
    P.close()


@pytest.mark.parametrize("alpha", [0.6, 0.7, 0.4, 1.3, 3.0, 0.05, 7.5, 0.5, 2.0])
def test_priority_alpha_keys(torch_cuda, alpha):
    """PER exponent (Q7): keys Q_F(RN(p^alpha)) made on the GPU (double-double
    exp/log, kernels/pow_dd.cuh) equal the oracle's (mpmath at 200 bits) for
    priorities spread over ~1e-20..1e20 plus edge values, through insert and
    through both update paths (fused and grid-wide); then sampling agrees."""
    cols = [synth.ColSpec("x", "u8", ())]
    N = 8192
    P = _pair(capacity=N, seq_len=1, colspecs=cols, R=2, alpha=alpha, max_batch=8192)
    rng = np.random.default_rng(int(alpha * 1000))
    p = np.exp(rng.normal(0.0, 10.0, N))
    p[::97] = 0.0
    edges = np.array([1.0, 2.0, 0.5, 2.0 ** -32, 2.0 ** 31, 1e-300, 1e300, 5e-324,
                      np.nextafter(1.0, 2.0), np.nextafter(1.0, 0.0), 3.0, 10.0, 0.1])
    p[:edges.size] = edges
    for s in range(2):
        P.insert(s, p[s * (N // 2):(s + 1) * (N // 2)])
    P.check_state()
    for fused in (1, 0):
        G.gear_table_set_tuning(P.t.handle, "update_fused", fused)
        ids = rng.permutation(N)[:4096].astype(np.uint64)
        q = np.exp(rng.normal(0.0, 6.0, ids.size))
        ost, ons, err, ns = P.update(ids, q)
        assert ost == 0 and err == 0
        P.check_state()
    P.check_sample(G.GEAR_PRIORITIZED, 512, 7, 0.4)
    P.close()


@pytest.mark.parametrize("removal", [0, 1])
@pytest.mark.parametrize("R", [1, 3])
def test_fifo_lifo_with_ring_wrap(torch_cuda, removal, R):
    """c4-style: each shard receives 1.25 x C_s inserts so the ring wraps;
    some trajectories are made unselectable; FIFO/LIFO selection must equal
    the oracle's global (seq, shard) order."""
    cols = [synth.ColSpec("obs", "f32", (4,)), synth.ColSpec("done", "u8", (3,))]
    Cs = 600
    P = _pair(capacity=Cs * R, seq_len=4, colspecs=cols, R=R, removal=removal)
    rng = np.random.default_rng(21)
    total = int(Cs * 1.25)
    for s in range(R):
        k = 0
        while k < total:
            b = int(rng.integers(1, 300))
            P.insert(s, np.ones(min(b, total - k)))
            k += b
    P.check_state()
    zero = rng.choice(Cs * R, size=Cs * R // 5, replace=False).astype(np.uint64)
    P.update(zero, np.zeros(zero.size))
    for B in (1, 7, 64, 200):
        for strat in (G.GEAR_FIFO, G.GEAR_LIFO):
            idx = P.check_sample(strat, B, 0)
            if idx is not None:
                P.check_collect(idx)
    P.check_sample(G.GEAR_FIFO, 4096, 0)  # more than selectable -> EMPTY
    P.close()


@pytest.mark.parametrize("R", [1, 3])
def test_topk_with_ties(torch_cuda, R):
    """TopK (Q20) on keys with many ties (priorities drawn
    from 7 values) and zeros, several K including the all-selectable and the
    EMPTY cases, a shard larger than one 1024-key chunk."""
    cols = [synth.ColSpec("x", "u8", (4,))]
    Cs = 2500
    P = _pair(capacity=Cs * R, seq_len=1, colspecs=cols, R=R)
    rng = np.random.default_rng(31)
    vals = np.array([0.0, 0.25, 0.5, 1.0, 2.0, 3.0, 1e-3])
    P.fill(vals[rng.integers(0, len(vals), size=Cs * R)])
    sel = int((P.o.key > 0).sum())
    for B in (1, 5, 64, 700, min(sel // 2, 4096)):
        idx = P.check_sample(G.GEAR_TOPK, B, 0)
        assert idx is not None
        P.check_collect(idx)
    ids = np.arange(0, Cs * R, 7, dtype=np.uint64)
    P.update(ids, rng.lognormal(0, 1, ids.size))
    P.check_sample(G.GEAR_TOPK, 333, 0)
    # few selectable: all of them, then one more than there are -> EMPTY
    P.update(np.arange(Cs * R, dtype=np.uint64)[:3000], np.zeros(3000))
    left = int((P.o.key > 0).sum())
    if left <= 4096:
        assert P.check_sample(G.GEAR_TOPK, left, 0) is not None
    if left + 1 <= 4096:
        assert P.check_sample(G.GEAR_TOPK, left + 1, 0) is None
    P.close()


@pytest.mark.parametrize("Cs", [120_000, 65_000, 60_000])
@pytest.mark.parametrize("R,kind", [(1, "ties"), (1, "lognormal"), (3, "ties"), (2, "equal")])
def test_topk_large_multi_cta(torch_cuda, R, kind, Cs):
    """TopK over shards spread across many CTAs per shard at the maximum
    K = 8192: ties straddling CTA slices, continuous keys (early exit of the
    select), and every key equal (the K taken are the K smallest slots).
    120 K / 65 K keys per shard take the grid-wide path (radix histograms
    merged in global memory), 60 K keys the cluster path (histograms merged
    through distributed shared memory)."""
    cols = [synth.ColSpec("x", "u8", (8,))]
    P = _pair(capacity=Cs * R, seq_len=1, colspecs=cols, R=R, max_batch=8192)
    rng = np.random.default_rng(77 + R)
    if kind == "ties":
        vals = np.array([0.0, 0.5, 1.0, 2.0, 4.0])
        prio = vals[rng.integers(0, len(vals), size=Cs * R)]
    elif kind == "lognormal":
        prio = synth.priorities(Cs * R, seed=5, zero_frac=0.05)
    else:
        prio = np.full(Cs * R, 1.5)
    P.fill(prio)
    for B in (1, 777, 8192):
        idx = P.check_sample(G.GEAR_TOPK, B, 0)
        assert idx is not None
    P.check_collect(idx)
    P.close()


@pytest.mark.parametrize("R,kind,B", [(1, "ties", 32768), (1, "lognormal", 100_000),
                                      (3, "ties", 20_000), (2, "equal", 7000)])
def test_topk_beyond_8192(torch_cuda, R, kind, B):
    """TopK with more candidates than the direct rank sort takes (K + 2048 >
    8192): sorted runs of 4096 candidates + merge ranks by binary search
    (topk.cu), up to 25 runs; ties across runs, every key equal (the K
    smallest slots), K at c5's W=8 batch (32768)."""
    cols = [synth.ColSpec("x", "u8", (4,))]
    Cs = 150_000
    P = _pair(capacity=Cs * R, seq_len=1, colspecs=cols, R=R, max_batch=B)
    rng = np.random.default_rng(B + R)
    if kind == "ties":
        vals = np.array([0.0, 0.5, 1.0, 2.0, 4.0])
        prio = vals[rng.integers(0, len(vals), size=Cs * R)]
    elif kind == "lognormal":
        prio = synth.priorities(Cs * R, seed=6, zero_frac=0.05)
    else:
        prio = np.full(Cs * R, 1.5)
    P.fill(prio)
    for b in (B, B - 4097):
        idx = P.check_sample(G.GEAR_TOPK, b, 0)
        assert idx is not None
    P.check_collect(idx)
    P.close()


def test_insert_bad_priority_and_device_sources(torch_cuda):
    cols = [synth.ColSpec("a", "u8", (7,)), synth.ColSpec("b", "i32", (3,))]
    P = _pair(capacity=64, seq_len=3, colspecs=cols, R=2)
    with pytest.raises(G.GearError) as e:
        P.t.insert(0, [np.zeros((2, P.rb[0]), np.uint8), np.zeros((2, P.rb[1]), np.uint8)],
                   np.array([1.0, np.nan]))
    assert e.value.status == G.GEAR_ERR_BAD_PRIORITY
    P.insert(0, np.linspace(0, 3, 32), device_src=True)
    P.insert(1, np.linspace(1, 2, 40), device_src=True)    # wraps shard 1 (C_s = 32)
    P.check_state()
    P.check_collect(np.arange(64, dtype=np.uint64))
    P.close()


def test_collect_index_range_latched(torch_cuda):
    cols = [synth.ColSpec("a", "u8", (16,))]
    P = _pair(capacity=32, seq_len=1, colspecs=cols)
    P.insert(0, np.ones(32))
    P.collect_gpu(np.array([1, 40, 3], np.uint64))
    err, _ = P.t.sync()
    assert err & G.GEAR_DEVERR_INDEX_RANGE
    P.close()


def test_figure4_collect_two_shards(torch_cuda):
    """collect([2, 4, 25, 26], [col0, col1]) over two shards of
    capacity 24 returns the rows in request order."""
    cols = [synth.ColSpec("col0", "f32", (3,)), synth.ColSpec("col1", "i32", ())]
    P = _pair(capacity=48, seq_len=2, colspecs=cols, R=2)
    P.insert(0, np.ones(24))
    P.insert(1, np.ones(24))
    P.check_collect(np.array([2, 4, 25, 26], np.uint64))
    P.close()


def test_host_buffers_through_abi(torch_cuda):
    """The C-ABI accepts host ids / priorities / sample outputs (pinned or
    pageable) and must give the same results as device buffers."""
    import torch
    P = _pair(capacity=C1.capacity, seq_len=C1.seq_len, colspecs=C1.cols, R=1)
    P.fill(synth.priorities(C1.capacity, seed=2, zero_frac=0.1))
    B = 64
    for pinned in (False, True):
        idx = torch.empty(B, dtype=torch.int64, pin_memory=pinned)
        w = torch.empty(B, dtype=torch.float32, pin_memory=pinned)
        P.t.sample(G.GEAR_PRIORITIZED, B, 77, 0.5, idx, w)
        torch.cuda.synchronize()
        st, oi, ow, op = P.sample_oracle(G.GEAR_PRIORITIZED, B, 77, 0.5)
        assert np.array_equal(idx.numpy().view(np.uint64), oi)
        np.testing.assert_allclose(w.numpy(), ow, rtol=1e-6)
        hp = torch.from_numpy(np.linspace(0.5, 2, B))
        hp = hp.pin_memory() if pinned else hp
        G.gear_update_priorities(P.t.handle, B, idx, hp, G.GEAR_F64)
        torch.cuda.synchronize()
        P.o.update(oi, np.linspace(0.5, 2, B))
        P.check_state()
    P.close()


def test_owner_affine_single_rank_is_identity(torch_cuda):
    """With one rank every entry is local: the owner-affine slice equals the
    contiguous one (the W>1 cases run in dist_gpu_parity.py)."""
    P = _pair(capacity=C1.capacity, seq_len=C1.seq_len, colspecs=C1.cols, R=4)
    P.fill(synth.priorities(C1.capacity, seed=6, zero_frac=0.1))
    for strat in (G.GEAR_UNIFORM, G.GEAR_WEIGHTED, G.GEAR_PRIORITIZED, G.GEAR_FIFO, G.GEAR_LIFO):
        a = P.sample_gpu(strat, 64, 17, 0.4)
        b = P.sample_gpu(strat | G.GEAR_SAMPLE_OWNER_AFFINE, 64, 17, 0.4)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        from gpu_harness import ORACLE_STRATEGY
        st, oi, ow, _ = P.o.sample(ORACLE_STRATEGY[strat], 1, 0, 64, 17, 0.4, owner_affine=True)
        assert st == 0 and np.array_equal(b[0], oi)
    P.close()


def test_deterministic_across_repeats_and_beta(torch_cuda):
    P = _pair(capacity=C1.capacity, seq_len=C1.seq_len, colspecs=C1.cols, R=4)
    P.fill(synth.priorities(C1.capacity, seed=5))
    a = P.sample_gpu(G.GEAR_PRIORITIZED, 512, 3, 0.0)
    b = P.sample_gpu(G.GEAR_PRIORITIZED, 512, 3, 1.0)
    assert np.array_equal(a[0], b[0])
    assert np.all(a[1] == 1.0)
    key = P.o.key[a[0].astype(np.int64)]
    qmin = key.min()
    assert np.array_equal(b[1], np.array([np.float32(int(qmin) / int(k)) for k in key]))
    P.check_sample(G.GEAR_PRIORITIZED, 512, 3, 1.0)
    P.close()


@pytest.mark.parametrize("impl,host_lsu", [(0, 1), (1, 1), (1, 0), (1, -1)])
@pytest.mark.parametrize("placement", ["device", "host"])
def test_collect_large_rows_tma_and_lsu(torch_cuda, impl, host_lsu, placement):
    """Rows >= 4 KB with 16-byte alignment take the TMA bulk-copy path
    (impl 1; host-resident ones by that kernel's LSU warps unless host_lsu is
    0), the rest the warp-LSU path; ragged last chunks, duplicate ids, three
    shards, both placements, several chunk sizes."""
    cols = [synth.ColSpec("big", "u8", (5008,)), synth.ColSpec("tok", "i32", (256,)),
            synth.ColSpec("odd", "u8", (7,)), synth.ColSpec("f", "f32", (3,))]
    P = _pair(capacity=3 * 97, seq_len=9, colspecs=cols, R=3, placement=placement)
    assert P.rb == [45072, 9216, 63, 108]
    P.fill(synth.priorities(3 * 97, seed=8))
    rng = np.random.default_rng(impl)
    G.gear_table_set_tuning(P.t.handle, "collect_impl", impl)
    G.gear_table_set_tuning(P.t.handle, "collect_host_lsu", host_lsu)
    for tma_chunk, lsu_chunk in ((32768, 8192), (4096, 512), (16384, 1024)):
        G.gear_table_set_tuning(P.t.handle, "tma_chunk", tma_chunk)
        G.gear_table_set_tuning(P.t.handle, "lsu_chunk", lsu_chunk)
        idx = rng.integers(0, 3 * 97, size=300).astype(np.uint64)
        P.check_collect(idx)
        P.check_collect(idx[:1], col_ids=[1, 0])
    with pytest.raises(G.GearError):
        G.gear_table_set_tuning(P.t.handle, "tma_chunk", 100)
    P.close()


@pytest.mark.parametrize("levels", [2, 1])
@pytest.mark.parametrize("R", [1, 3, 8])
def test_adversarial_keys(torch_cuda, R, levels):
    """SURVEY.md §8 d.1 extras: every key at q_max (the total just below 2^62),
    one dominant q_max key among keys of 1, and a single selectable slot --
    sampled ids, q/T and IS weights equal the oracle's on both CDF layouts."""
    cols = [synth.ColSpec("x", "u8", (2,))]
    Cs = 4096 + 123                                    # two tiles per shard, ragged
    N = Cs * R
    P = _pair(capacity=N, seq_len=1, colspecs=cols, R=R)
    G.gear_table_set_tuning(P.t.handle, "cdf_levels", levels)
    P.fill(np.full(N, 1e300))                          # all keys q_max: T = N*q_max < 2^62
    qmax = G.gear_table_info_get(P.t.handle)["q_max"]
    assert int(P.o.key.astype(object).sum()) == N * qmax < (1 << 62)
    for strat in (G.GEAR_PRIORITIZED, G.GEAR_WEIGHTED, G.GEAR_UNIFORM):
        P.check_sample(strat, 2048, 11, beta=0.7)
    ids = np.arange(N, dtype=np.uint64)

    def update_all(v):                                 # in max_batch chunks
        for k0 in range(0, N, 4096):
            P.update(ids[k0:k0 + 4096], np.full(min(4096, N - k0), v))

    update_all(2.0 ** -32)                             # every key 1 ...
    P.update(np.array([N // 2 + 7], np.uint64), [1e300])   # ... but one at q_max
    P.check_state()
    idx = P.check_sample(G.GEAR_PRIORITIZED, 2048, 12, beta=0.4)
    assert np.mean(idx == N // 2 + 7) > 0.9
    update_all(0.0)                                    # nothing selectable but one
    P.update(np.array([N - 1], np.uint64), [3.0])
    for strat in (G.GEAR_PRIORITIZED, G.GEAR_UNIFORM, G.GEAR_FIFO, G.GEAR_TOPK):
        if strat in (G.GEAR_FIFO, G.GEAR_TOPK):
            idx = P.check_sample(strat, 1, 0)
        else:
            idx = P.check_sample(strat, 512, 13)
        assert np.all(idx == N - 1)
    P.update(np.array([N - 1], np.uint64), [0.0])      # nothing selectable: EMPTY
    assert P.check_sample(G.GEAR_PRIORITIZED, 64, 14) is None
    P.close()


def test_update_from_pinned_and_pageable_host(torch_cuda):
    """gear_update_priorities reads pinned host ids / priorities / generations
    in place (zero-copy) and copies pageable ones; both equal the oracle."""
    torch = torch_cuda
    cols = [synth.ColSpec("x", "u8", (4,))]
    P = _pair(capacity=512, seq_len=1, colspecs=cols, R=2)
    P.fill(np.ones(512))
    rng = np.random.default_rng(3)
    for kind in ("pinned", "pageable"):
        for fused in (1, 0):
            G.gear_table_set_tuning(P.t.handle, "update_fused", fused)
            ids = rng.integers(0, 512, 300).astype(np.uint64)
            p = rng.lognormal(0, 1, 300)
            gen = P.o.gen[ids.astype(np.int64)].copy()
            gen[::5] += 1                                   # some stale
            if kind == "pinned":
                h_ids = torch.from_numpy(ids.view(np.int64)).pin_memory()
                h_p = torch.from_numpy(p).pin_memory()
                h_g = torch.from_numpy(gen.view(np.int32)).pin_memory()
            else:
                h_ids, h_p, h_g = ids, p, gen
            G.gear_update_priorities(P.t.handle, 300, h_ids, h_p, G.GEAR_F64, h_g)
            torch.cuda.synchronize()
            ost, ons = P.o.update(ids, p, gen)
            err, ns = P.t.sync()
            assert ns == ons
            P.check_state()
    P.close()


@pytest.mark.parametrize("strat", ["prioritized", "fifo"])
def test_sample_into_pinned_and_pageable_host(torch_cuda, strat):
    """gear_sample writes pinned host outputs in place (mapped, zero-copy) and
    pageable ones through scratch + copy; both equal the device outputs and
    the oracle."""
    torch = torch_cuda
    import oracle
    cols = [synth.ColSpec("x", "u8", (4,))]
    P = _pair(capacity=600, seq_len=1, colspecs=cols, R=3)
    P.fill(synth.priorities(600, seed=8, zero_frac=0.1))
    S = G.GEAR_PRIORITIZED if strat == "prioritized" else G.GEAR_FIFO
    B = 200
    st, oi, ow, op = P.o.sample(oracle.PRIORITIZED if strat == "prioritized" else oracle.FIFO,
                                1, 0, B, 77, 0.4)
    assert st == 0
    pin = [torch.empty(B, dtype=d).pin_memory() for d in (torch.int64, torch.float32,
                                                          torch.float64, torch.int32)]
    G.gear_sample(P.t.handle, S, B, 77, 0.4, *pin)
    torch.cuda.synchronize()
    pag = [np.empty(B, np.uint64), np.empty(B, np.float32), np.empty(B, np.float64),
           np.empty(B, np.uint32)]
    G.gear_sample(P.t.handle, S, B, 77, 0.4, *pag)
    torch.cuda.synchronize()
    for out in (pin, pag):
        idx = out[0].numpy().view(np.uint64) if hasattr(out[0], "numpy") else out[0]
        w = out[1].numpy() if hasattr(out[1], "numpy") else out[1]
        p = out[2].numpy() if hasattr(out[2], "numpy") else out[2]
        assert np.array_equal(idx, oi)
        np.testing.assert_allclose(w, ow, rtol=1e-6, atol=0)
        assert np.array_equal(p, op)
    assert P.t.sync()[0] == 0
    P.close()


def test_host_rows_straddling_registration_pieces(torch_cuda, monkeypatch):
    """Host columns are registered with CUDA in pieces (api.cpp map_host; 64 GiB
    by default, 2 MiB here): rows that straddle two pieces are inserted and
    collected byte-exactly, on the LSU path (3000-B rows) and the TMA bulk path
    (12000-B rows)."""
    monkeypatch.setenv("GEAR_HOST_REG_CHUNK", str(2 << 20))
    cols = [synth.ColSpec("a", "u8", (1000,), "host"), synth.ColSpec("b", "i32", (1000,), "host")]
    N = 1500
    P = _pair(capacity=N, seq_len=3, colspecs=cols)
    assert P.rb == [3000, 12000]
    P.fill(synth.priorities(N, seed=5))
    straddle = [g for g in range(N) for rb in P.rb
                if (g * rb) // (2 << 20) != ((g + 1) * rb - 1) // (2 << 20)]
    assert len(straddle) > 8
    P.check_collect(np.asarray(sorted(set(straddle)), np.uint64))
    P.check_collect(np.random.default_rng(3).permutation(N).astype(np.uint64))
    P.check_collect(P.check_sample(G.GEAR_WEIGHTED, 1024, 77))
    P.close()


def test_zero_size_calls_are_noops(torch_cuda):
    """B = 0 / n = 0 (include/gear.h): sample, collect and update return OK
    without touching their outputs or the table, and without advancing the
    device seed counter -- the next draw still equals the oracle's."""
    import oracle
    torch = torch_cuda
    cols = [synth.ColSpec("x", "f32", (2,))]
    P = _pair(capacity=4096, seq_len=1, colspecs=cols, R=2)
    P.fill(synth.priorities(4096, seed=3, zero_frac=0.05))
    h = P.t.handle
    idx = torch.full((8,), 7, dtype=torch.int64, device="cuda")
    w = torch.full((8,), 3.0, dtype=torch.float32, device="cuda")
    out = torch.full((8, P.rb[0]), 0xAB, dtype=torch.uint8, device="cuda")
    G.gear_table_set_tuning(h, "device_seed", 0x5EED)
    for strat in (G.GEAR_UNIFORM, G.GEAR_PRIORITIZED, G.GEAR_FIFO, G.GEAR_TOPK):
        G.gear_sample(h, strat, 0, 0, 0.4, idx, w, flags=G.GEAR_SAMPLE_DEVICE_SEED)
    G.gear_collect(h, 0, idx, [0], [out])
    G.gear_update_priorities(h, 0, idx, torch.zeros(8, dtype=torch.float64, device="cuda"),
                             G.GEAR_F64)
    torch.cuda.synchronize()
    assert torch.all(idx == 7) and torch.all(w == 3.0) and torch.all(out == 0xAB)
    err, stale = P.t.sync()
    assert err == 0 and stale == 0
    P.check_state()
    # the seed counter did not move: the first real draw uses seed 0x5EED
    G.gear_sample(h, G.GEAR_PRIORITIZED, 8, 0, 0.4, idx, w, flags=G.GEAR_SAMPLE_DEVICE_SEED)
    torch.cuda.synchronize()
    st, oi, ow, _ = P.o.sample(oracle.PRIORITIZED, 1, 0, 8, 0x5EED, 0.4)
    assert st == 0
    assert np.array_equal(idx.cpu().numpy().view(np.uint64), oi)
    np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-6, atol=0)
    P.close()


@pytest.mark.parametrize("R", [1, 3])
def test_max_batch_one_million(torch_cuda, R):
    """A batch at the top of the size range (B = 2^20, W * max_batch < 2^24):
    ids, IS weights, q/T and every collected row of a 2^20-row prioritized
    and uniform draw, then a 2^20-entry update with duplicates, then FIFO and
    LIFO at 2^20 (more candidates than one merge tile)."""
    cols = [synth.ColSpec("x", "u8", (12,))]
    B = 1 << 20
    N = R * 700_001
    P = _pair(capacity=N, seq_len=1, colspecs=cols, R=R, max_batch=B)
    P.fill(synth.priorities(N, seed=9, zero_frac=0.1))
    for strat, seed in ((G.GEAR_PRIORITIZED, 77), (G.GEAR_UNIFORM, 78)):
        idx = P.check_sample(strat, B, seed)
        P.check_collect(idx)
    rng = np.random.default_rng(5)
    ost, _, err, _ = P.update(idx, rng.lognormal(0, 1, B))
    assert ost == 0 and err == 0
    P.check_state()
    P.check_sample(G.GEAR_PRIORITIZED, B, 79)
    for strat in (G.GEAR_FIFO, G.GEAR_LIFO):
        P.check_sample(strat, B // 2, 80)
    P.close()
