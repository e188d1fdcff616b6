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


def test_device_priorities_rejected_on_device(torch_cuda):
    """gear_insert with device priorities validates them on the device: a NaN
    latches BAD_PRIORITY and nothing is inserted."""
    torch = torch_cuda
    cols = [synth.ColSpec("x", "u8", (4,))]
    P = _pair(capacity=64, seq_len=1, colspecs=cols, R=1)
    P.insert(0, np.ones(10))
    src = [torch.zeros((3, P.rb[0]), dtype=torch.uint8, device="cuda")]
    prio = torch.tensor([1.0, float("nan"), 2.0], dtype=torch.float64, device="cuda")
    out = torch.empty(3, dtype=torch.int64, device="cuda")
    P.t.insert(0, src, prio, out)
    err, _ = P.t.sync()
    assert err & G.GEAR_DEVERR_BAD_PRIORITY
    assert np.all(out.cpu().numpy().view(np.uint64) == np.uint64(G.GEAR_IDX_NONE))
    P.check_state()
    P.insert(0, np.ones(5))            # the allocator state was not touched
    P.check_state()
    P.close()


@pytest.mark.parametrize("removal", [0, 1])
def test_writer_calls_captured_in_a_graph(torch_cuda, removal):
    """gear_insert (device rows and priorities) and gear_allocate -> gear_commit
    (ids flowing through device memory) captured once in a CUDA graph and
    replayed: every replay runs the allocator again on the device state and
    equals the oracle doing the same calls."""
    torch = torch_cuda
    import oracle
    cols = [synth.ColSpec("obs", "f32", (5,)), synth.ColSpec("act", "i32", ())]
    Cs, B, A = 200, 48, 30
    P = _pair(capacity=Cs, seq_len=2, colspecs=cols, R=1, removal=removal)
    P.insert(0, synth.priorities(120, seed=1))
    traj = np.arange(50_000, 50_000 + B)
    rows = [synth.row_bytes_of(c, traj, rb) for c, rb in enumerate(P.rb)]
    srcs = [torch.from_numpy(r).cuda() for r in rows]
    p_ins = synth.priorities(B, seed=2)
    p_com = synth.priorities(A, seed=3)
    d_pins = torch.from_numpy(p_ins).cuda()
    d_pcom = torch.from_numpy(p_com).cuda()
    out_ins = torch.empty(B, dtype=torch.int64, device="cuda")
    out_al = torch.empty(A, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s, capture_error_mode="thread_local"):
        G.gear_insert(P.t.handle, 0, B, srcs, d_pins, out_ins, s)
        G.gear_allocate(P.t.handle, 0, A, out_al, s)
        G.gear_commit(P.t.handle, 0, A, out_al, d_pcom, s)
    torch.cuda.synchronize()
    P.check_state()                    # capturing ran nothing
    for rep in range(6):
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        st, oids = P.o.insert(0, p_ins)
        assert st == 0
        for c in range(len(P.rb)):
            P.mirror[c][oids.astype(np.int64)] = rows[c]
        st, aids = P.o.allocate(0, A)
        assert st == 0
        assert P.o.commit(0, aids, p_com) == 0
        assert np.array_equal(out_ins.cpu().numpy().view(np.uint64), oids)
        assert np.array_equal(out_al.cpu().numpy().view(np.uint64), aids)
        P.t.sync()
        P.check_state()
        for strat in (G.GEAR_FIFO, G.GEAR_LIFO, G.GEAR_PRIORITIZED):
            idx = P.check_sample(strat, 64, rep)
            P.check_collect(idx)
    assert oracle.OK == 0
    P.close()
