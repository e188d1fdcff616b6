"""K1 CDF kernels against the oracle's CDF ("computes a prefix
sum array using the decoupled look-back algorithm"): EVERY entry of every
local shard's CDF -- the flat decoupled look-back scan (cdf_levels 1) and the
two-level incremental layout (cdf_levels 2), weights and indicator mode --
equals oracle.cdf (gor_cdf, the sequential u64 sum) of the same keys, at
sizes whose shards span hundreds of 4096-key tiles (more than the 128-tile
look-back window) with a ragged last tile, after full builds and after
sparse updates."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


def _check_cdf(P, R, Cs, indicator):
    import oracle
    import paper_2310_05205_b200 as G
    got = G.gear_read_cdf(P.t.handle)
    key = P.o.key
    for ls in range(R):
        k = key[ls * Cs:(ls + 1) * Cs]
        want = oracle.cdf((k > 0).astype(np.uint64) if indicator else k)
        g = got[ls * Cs:(ls + 1) * Cs]
        if not np.array_equal(g, want):
            bad = np.nonzero(g != want)[0]
            raise AssertionError(f"shard {ls}: {bad.size} CDF entries differ, first at {bad[:5]} "
                                 f"(tile {bad[0] // 4096})")


# (cdf_levels, scan_chunk): the flat look-back over 4096-key tiles (chunk 0),
# over one chunk per CTA (chunk 1), over chunks with the grid capped at 7 CTAs
# so every CTA claims several chunks (chunk 7), and the two-level layout
LAYOUTS = [(1, 0), (1, 1), (1, 7), (2, -1)]


@pytest.mark.parametrize("levels,chunk", LAYOUTS)
@pytest.mark.parametrize("R,Cs", [(1, 3_000_017), (3, 700_001), (8, 150_003)])
def test_cdf_every_entry(torch_cuda, levels, chunk, R, Cs):
    import paper_2310_05205_b200 as G
    from gpu_harness import Pair
    P = Pair(capacity=Cs * R, seq_len=1, colspecs=[synth.ColSpec("x", "u8", (1,))], R=R,
             mirror=False)
    G.gear_table_set_tuning(P.t.handle, "cdf_levels", levels)
    G.gear_table_set_tuning(P.t.handle, "scan_chunk", chunk)
    prio = synth.priorities(Cs * R, seed=11, zero_frac=0.05)
    for s in range(R):
        P.t.insert(s, [np.zeros((Cs, 1), np.uint8)], prio[s * Cs:(s + 1) * Cs])
        P.o.insert(s, prio[s * Cs:(s + 1) * Cs])
    rng = np.random.default_rng(levels)
    for rnd in range(4):
        P.check_sample(G.GEAR_PRIORITIZED, 4096, 77 + rnd)
        _check_cdf(P, R, Cs, indicator=False)
        P.check_sample(G.GEAR_UNIFORM, 1024, 99 + rnd)
        _check_cdf(P, R, Cs, indicator=True)
        ids = rng.integers(0, Cs * R, 4096).astype(np.uint64)
        p = rng.lognormal(0, 2, ids.size) * (rng.random(ids.size) > 0.1)
        if rnd == 2:
            p[:] = 1e300                         # every updated key saturates at q_max
        P.update(ids, p)
    P.close()


def test_cdf_layout_switches(torch_cuda):
    """Flat and two-level builds interleaved on one table (they share the
    CDF double buffer and its parity; the flat scan's status arrays alternate
    by their own epoch): every build's CDF equals the oracle's, with updates
    between builds."""
    import paper_2310_05205_b200 as G
    from gpu_harness import Pair
    R, Cs = 2, 1_100_000
    P = Pair(capacity=Cs * R, seq_len=1, colspecs=[synth.ColSpec("x", "u8", (1,))], R=R,
             mirror=False)
    prio = synth.priorities(Cs * R, seed=5, zero_frac=0.02)
    for s in range(R):
        P.t.insert(s, [np.zeros((Cs, 1), np.uint8)], prio[s * Cs:(s + 1) * Cs])
        P.o.insert(s, prio[s * Cs:(s + 1) * Cs])
    rng = np.random.default_rng(9)
    seq = [(1, 0), (1, 1), (2, -1), (1, 0), (2, -1), (2, -1), (1, 1), (1, 0), (1, 1), (1, 5)]
    for rnd, (levels, chunk) in enumerate(seq):
        G.gear_table_set_tuning(P.t.handle, "cdf_levels", levels)
        G.gear_table_set_tuning(P.t.handle, "scan_chunk", chunk)
        P.check_sample(G.GEAR_PRIORITIZED, 2048, 300 + rnd)
        _check_cdf(P, R, Cs, indicator=False)
        ids = rng.integers(0, Cs * R, 512).astype(np.uint64)
        P.update(ids, rng.lognormal(0, 1, ids.size))
    P.close()
