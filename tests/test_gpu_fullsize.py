"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (bench.build_table + the bench step): the oracle recomputes every
sampled id of every step (its CDF over all N keys), the IS weights, the keys
after the step's update, and EVERY collected row of EVERY column is compared
byte for byte with the expected batch -- the rows of the oracle's ids
regenerated on the GPU by the seeded row generator (synth.fill_rows_ids, the
same splitmix64 stream numpy computes; pinned to numpy by
test_synth_fill_matches_numpy), so no second copy of a 85 GB table is needed
(the collected rows "concatenated" in request order).

Tables whose host columns exceed the box's RAM (c4, c5) are scaled to the
largest N bench.scaled_capacity fits; the row layout is the config's.
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


def test_synth_fill_matches_numpy(torch_cuda):
    """The GPU row generator equals the numpy one (ragged row sizes, ids
    spanning 2^32, row_bytes not a multiple of 8)."""
    import synth
    torch = torch_cuda
    ids = np.array([0, 1, 7, 99_999, 2 ** 32 + 5, 10 ** 7 - 1], np.uint64)
    d_ids = torch.from_numpy(ids.view(np.int64)).cuda()
    for col, rb in ((0, 8), (1, 120), (2, 847_080 - 360), (3, 13), (5, 1)):
        out = torch.empty((ids.size, rb), dtype=torch.uint8, device="cuda")
        synth.fill_rows_ids(out.data_ptr(), d_ids.data_ptr(), ids.size, rb, col)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), synth.row_bytes_of(col, ids, rb)), (col, rb)
        first = torch.empty((3, rb), dtype=torch.uint8, device="cuda")
        synth.fill_rows(first.data_ptr(), 3, rb, col, 41)
        torch.cuda.synchronize()
        assert np.array_equal(first.cpu().numpy(), synth.row_bytes_of(col, [41, 42, 43], rb))


def _check_batch(torch, outs, row_bytes, oi, stream, what):
    """Every row of every column equals the regenerated row of the oracle's
    id (slot g holds trajectory g: bench.build_table inserts in id order)."""
    import synth
    d_ids = torch.from_numpy(oi.view(np.int64)).cuda()
    for c, rb in enumerate(row_bytes):
        want = torch.empty_like(outs[c])
        with torch.cuda.stream(stream):
            synth.fill_rows_ids(want.data_ptr(), d_ids.data_ptr(), len(oi), rb, c,
                                stream=stream.cuda_stream)
        stream.synchronize()
        if not torch.equal(outs[c], want):
            bad = (outs[c] != want).any(dim=1).nonzero().flatten()[:8].tolist()
            raise AssertionError(f"{what}: column {c} rows differ at {bad}")


def _run_config(torch, name, phases):
    """phases: [(strategy or None, update, steps)] on ONE full-size table."""
    import dataclasses
    import bench
    import oracle
    import synth
    import paper_2310_05205_b200 as gear
    base = synth.CONFIGS[name]
    capacity, note = bench.scaled_capacity(base, 1)
    stream = torch.cuda.Stream()
    t, prio_all = bench.build_table(base, None, 1, 0, capacity, stream)
    o = oracle.Table(capacity, 1)
    o.insert(0, prio_all)
    key, _, _ = t.read_state()
    assert np.array_equal(key, o.key)
    B = base.batch
    idx = torch.empty(B, dtype=torch.int64, device="cuda")
    w = torch.empty(B, dtype=torch.float32, device="cuda")
    outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
    ostrats = {"prioritized": oracle.PRIORITIZED, "weighted": oracle.WEIGHTED,
               "fifo": oracle.FIFO, "lifo": oracle.LIFO, "topk": oracle.TOPK}
    step = 0
    for strategy, update, steps in phases:
        cfg = dataclasses.replace(base, strategy=strategy or base.strategy, update=update)
        strat = gear.STRATEGIES[cfg.strategy]
        for _ in range(steps):
            seed = synth.SAMPLE_SEED_BASE + step
            gear.gear_sample(t.handle, strat, B, seed, cfg.beta, idx, w, None, None, stream)
            gear.gear_collect(t.handle, B, idx, list(range(len(outs))), outs, stream)
            p = synth.priorities(B, seed=1000 + step)
            if cfg.update:
                gear.gear_update_priorities(t.handle, B, idx, torch.from_numpy(p).cuda(),
                                            gear.GEAR_F64, None, stream)
            stream.synchronize()
            st, oi, ow, _ = o.sample(ostrats[cfg.strategy], 1, 0, B, seed, cfg.beta)
            assert st == 0
            gi = idx.cpu().numpy().view(np.uint64)
            assert np.array_equal(gi, oi), f"{name} {cfg.strategy} step {step}: ids differ"
            np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-6, atol=0)
            _check_batch(torch, outs, t.row_bytes, oi, stream, f"{name} {cfg.strategy} step {step}")
            if cfg.update:
                o.update(oi, p)
            step += 1
    key, _, _ = t.read_state()
    assert np.array_equal(key, o.key)
    err, _ = t.sync()
    assert err == 0
    t.close()
    print(f"{name}: N={capacity} ({note or 'full size'}), {step} steps x {B} rows x "
          f"{sum(t.row_bytes)} B compared byte for byte")
    return capacity, note


def test_c2_full_size_hbm(torch_cuda):
    """c2 at 100,000 x 847,080 B (84.7 GB HBM): every row of 4 steps."""
    _run_config(torch_cuda, "c2", [(None, True, 4)])


def test_c3_full_size_host(torch_cuda):
    """c3 at 1,000,000 x 4,096 B host-pinned: every row of 3 steps."""
    _run_config(torch_cuda, "c3", [(None, False, 3)])


def test_c5_host_largest_fit(torch_cuda):
    """c5 at the largest N that fits 60% of host RAM: every row of 2
    prioritized steps with updates."""
    _run_config(torch_cuda, "c5", [(None, True, 2)])


def test_c4_mixed_prioritized_fifo_lifo_topk(torch_cuda):
    """c4 (HBM + host columns in one row) at the largest N that fits:
    prioritized with per-step updates, then FIFO, LIFO and TopK on the same
    table -- every row of every column of every step."""
    _run_config(torch_cuda, "c4", [(None, True, 3), ("fifo", False, 1), ("lifo", False, 1),
                                   ("topk", False, 1)])
