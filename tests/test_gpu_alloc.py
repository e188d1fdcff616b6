"""NEXT-1: the device-resident block allocator (kernels/alloc.cu) against the
oracle -- gear_allocate / rows written in place / gear_commit (PAPER.md:193,
reading Q21), gear_insert planned on the device, FIFO/LIFO removal, FULL,
stale updates to ongoing slots, selection and collection of what was
committed."""
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


def _pair(**kw):
    from gpu_harness import Pair
    return Pair(**kw)


G = __import__("paper_2310_05205_b200")


@pytest.mark.parametrize("placement", ["device", "host"])
@pytest.mark.parametrize("removal", [0, 1])
def test_allocate_commit_interleaved(torch_cuda, removal, placement):
    cols = [synth.ColSpec("obs", "f32", (6,)), synth.ColSpec("act", "u8", (5,))]
    R, Cs = 2, 40
    P = _pair(capacity=Cs * R, seq_len=3, colspecs=cols, R=R, removal=removal,
              placement=placement)
    rng = np.random.default_rng(100 + removal)
    pending = {0: [], 1: []}
    for step in range(70):
        s = int(rng.integers(0, R))
        op = int(rng.integers(0, 5))
        if op == 0:
            ids = P.allocate(s, int(rng.integers(1, 30)))
            if ids is not None:
                P.write_rows(ids)
                pending[s] += [int(x) for x in ids]
        elif op == 1 and pending[s]:
            k = int(rng.integers(1, len(pending[s]) + 1))
            ids = list(rng.permutation(pending[s])[:k])
            if rng.random() < 0.3:
                ids.append(ids[-1])                       # duplicate: second copy stale
            if rng.random() < 0.2:
                ids.append(int(rng.integers(0, Cs * R)))  # maybe another shard / not ongoing
            prio = synth.priorities(len(ids), seed=step, zero_frac=0.1)
            if rng.random() < 0.2:
                prio[0] = -1.0                            # bad priority: stays ongoing
            P.commit(s, ids, prio)
            o = P.o
            pending[s] = [g for g in pending[s] if o.seq[g] == 0 and o.gen[g] > 0]
        elif op == 2:
            P.insert(s, synth.priorities(int(rng.integers(1, 60)), seed=step))
            o = P.o
            pending[s] = [g for g in pending[s] if o.seq[g] == 0 and o.gen[g] > 0]
        elif op == 3:
            ids = rng.integers(0, Cs * R, 10).astype(np.uint64)
            ost, ons, err, ns = P.update(ids, rng.lognormal(0, 1, 10))
            assert ons == ns                              # ongoing / never inserted -> stale
        else:
            for strat in (G.GEAR_FIFO, G.GEAR_LIFO, G.GEAR_PRIORITIZED):
                idx = P.check_sample(strat, 16, step)
                if idx is not None:
                    P.check_collect(idx)
        P.check_state()
    P.close()


@pytest.mark.parametrize("removal", [0, 1])
def test_insert_plan_wraps_with_ongoing_slots(torch_cuda, removal):
    """One gear_insert call of many more rows than free + committed slots, with
    some slots held ongoing: the closed-form plan (slot k mod C, last row
    wins, ring position) equals the row-by-row oracle."""
    cols = [synth.ColSpec("x", "i32", (7,))]
    Cs = 300
    P = _pair(capacity=Cs, seq_len=2, colspecs=cols, R=1, removal=removal)
    P.insert(0, synth.priorities(200, seed=1))
    held = P.allocate(0, 37)                               # ongoing: not reusable
    P.write_rows(held)
    for n in (1, 63, 263, 1000, 2500):
        P.insert(0, synth.priorities(n, seed=n))
        P.check_state()
        for strat in (G.GEAR_FIFO, G.GEAR_LIFO):
            idx = P.check_sample(strat, 100, 0)
            if idx is not None:
                P.check_collect(idx)
    P.commit(0, held, np.linspace(0.5, 2.0, held.size))
    P.check_state()
    idx = P.check_sample(G.GEAR_LIFO, 50, 0)
    P.check_collect(idx)
    P.close()


def test_full_shard(torch_cuda):
    """Every slot ongoing: allocate and insert latch FULL and change nothing."""
    cols = [synth.ColSpec("x", "u8", (4,))]
    P = _pair(capacity=64, seq_len=1, colspecs=cols, R=1)
    ids = P.allocate(0, 64)
    assert ids is not None
    assert P.allocate(0, 1) is None
    import oracle
    P.t.insert(0, [np.zeros((1, 4), np.uint8)], np.ones(1))
    err, _ = P.t.sync()
    assert err & G.GEAR_DEVERR_FULL
    assert P.o.insert(0, np.ones(1))[0] == oracle.FULL
    P.check_state()
    P.write_rows(ids)
    P.commit(0, ids, np.ones(64))
    idx = P.check_sample(G.GEAR_FIFO, 64, 0)
    P.check_collect(idx)
    P.close()
