"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (bench.build_table + the bench step): the oracle recomputes every
sampled id of the step (its CDF over all N keys), the keys after the step's
update, and the bytes of a sample of the collected rows (regenerated from the
seeded row generator -- no second copy of a 85 GB table is needed)."""
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


def _run_config(torch, name, steps=3, rows_checked=24, strategy=None):
    import dataclasses
    import bench
    import oracle
    import synth
    import paper_2310_05205_b200 as gear
    cfg = synth.CONFIGS[name]
    if strategy:
        cfg = dataclasses.replace(cfg, strategy=strategy, update=False)
    capacity, note = bench.scaled_capacity(cfg, 1)
    stream = torch.cuda.Stream()
    t, prio_all = bench.build_table(cfg, None, 1, 0, capacity, stream)
    o = oracle.Table(capacity, 1)
    o.insert(0, prio_all)
    key, _, _ = t.read_state()
    assert np.array_equal(key, o.key)
    B = cfg.batch
    strat = gear.STRATEGIES[cfg.strategy]
    ostrat = {"prioritized": oracle.PRIORITIZED, "weighted": oracle.WEIGHTED,
              "fifo": oracle.FIFO, "lifo": oracle.LIFO}[cfg.strategy]
    idx = torch.empty(B, dtype=torch.int64, device="cuda")
    w = torch.empty(B, dtype=torch.float32, device="cuda")
    outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
    rng = np.random.default_rng(0)
    for i in range(steps):
        seed = synth.SAMPLE_SEED_BASE + i
        gear.gear_sample(t.handle, strat, B, seed, cfg.beta, idx, w, None, None, stream)
        gear.gear_collect(t.handle, B, idx, list(range(len(outs))), outs, stream)
        p = synth.priorities(B, seed=1000 + i)
        if cfg.update:
            gear.gear_update_priorities(t.handle, B, idx, torch.from_numpy(p).cuda(), gear.GEAR_F64,
                                        None, stream)
        stream.synchronize()
        st, oi, ow, _ = o.sample(ostrat, 1, 0, B, seed, cfg.beta)
        gi = idx.cpu().numpy().view(np.uint64)
        assert np.array_equal(gi, oi), f"{name} step {i}: ids differ"
        np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=1e-6)
        js = rng.choice(B, size=min(rows_checked, B), replace=False)
        for c, rb in enumerate(t.row_bytes):
            got = outs[c][torch.from_numpy(js).cuda()].cpu().numpy()
            want = synth.row_bytes_of(c, oi[js], rb)     # slot g holds trajectory g
            assert np.array_equal(got, want), f"{name} step {i}: column {c} rows differ"
        if cfg.update:
            o.update(oi, p)
    key, _, _ = t.read_state()
    assert np.array_equal(key, o.key)
    err, _ = t.sync()
    assert err == 0
    t.close()


def test_c2_full_size_hbm(torch_cuda):
    _run_config(torch_cuda, "c2")


def test_c3_full_size_host(torch_cuda):
    _run_config(torch_cuda, "c3")


def test_c5_host_scaled(torch_cuda):
    _run_config(torch_cuda, "c5", steps=2)


@pytest.mark.parametrize("strategy", ["fifo", "lifo"])
def test_c4_mixed_fifo_lifo_scaled(torch_cuda, strategy):
    """c4 (HBM + host columns), FIFO/LIFO over the whole table (N scaled to
    the box's host RAM)."""
    _run_config(torch_cuda, "c4", steps=2, strategy=strategy)
