"""Shard checkpoint / restore: a table saved after inserts
(with ring wrap) and priority updates and loaded into a fresh table of the
same layout continues exactly like the oracle: same keys/seq/gen, same
samples, same collected bytes, same FIFO order and slot assignment."""
import os

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


@pytest.mark.parametrize("placement", ["device", "host"])
def test_save_load_round_trip(torch_cuda, tmp_path, placement):
    import oracle
    import paper_2310_05205_b200 as G
    from gpu_harness import Pair
    cols = [synth.ColSpec("obs", "f32", (5,)), synth.ColSpec("tok", "i32", (300,))]
    Cs, R = 400, 2
    P = Pair(capacity=Cs * R, seq_len=4, colspecs=cols, R=R, placement=placement)
    for s in range(R):
        P.insert(s, synth.priorities(int(Cs * 1.3), seed=s, zero_frac=0.1))   # ring wraps
    P.update(np.arange(0, Cs * R, 3, dtype=np.uint64), synth.priorities(len(range(0, Cs * R, 3)), seed=9))
    path = str(tmp_path / f"shard_r0_{placement}.gear")
    P.t.save(path)
    assert os.path.getsize(path) > sum(P.rb) * Cs * R
    # a fresh table of the same layout
    Q = Pair(capacity=Cs * R, seq_len=4, colspecs=cols, R=R, placement=placement, mirror=False)
    Q.t.load(path)
    Q.o, Q.mirror, Q.content, Q.next_traj = P.o, P.mirror, P.content, P.next_traj
    Q.check_state()
    for strat in (G.GEAR_PRIORITIZED, G.GEAR_UNIFORM, G.GEAR_FIFO, G.GEAR_LIFO, G.GEAR_TOPK):
        idx = Q.check_sample(strat, 64, 123, 0.4)
        Q.check_collect(idx)
    # the restored rings keep allocating where the saved ones left off
    Q.insert(1, np.ones(50))
    Q.check_state()
    Q.check_sample(G.GEAR_FIFO, 100, 0)
    # a table of another layout refuses the file
    bad = Pair(capacity=Cs * R * 2, seq_len=4, colspecs=cols, R=R, mirror=False)
    with pytest.raises(G.GearError):
        bad.t.load(path)
    for x in (P, Q, bad):
        x.close()


def test_checkpoint_refusals(torch_cuda, tmp_path):
    """Save refuses an in-flight allocation (its slot would leak on restore)
    and leaves the previous checkpoint intact; load refuses another schema
    (same row bytes, renamed / retyped column) and a truncated file, and
    leaves the table unchanged."""
    import paper_2310_05205_b200 as G
    from gpu_harness import Pair
    torch = torch_cuda
    cols = [synth.ColSpec("obs", "f32", (4,)), synth.ColSpec("act", "i32", ())]
    Cs, R = 300, 2
    P = Pair(capacity=Cs * R, seq_len=3, colspecs=cols, R=R)
    for s in range(R):
        P.insert(s, synth.priorities(200, seed=s))
    path = str(tmp_path / "ck.gear")
    P.t.save(path)
    good = open(path, "rb").read()
    ids = P.allocate(0, 5)                      # in flight
    with pytest.raises(G.GearError) as e:
        P.t.save(path)
    assert e.value.status == G.GEAR_ERR_STATE
    assert open(path, "rb").read() == good and not os.path.exists(path + ".tmp")
    P.write_rows(ids)
    P.commit(0, ids, np.ones(5))
    P.t.save(path)                              # committed: saves again
    # same row bytes, another schema: f32[4] -> i32[4], and a renamed column
    for other in ([synth.ColSpec("obs", "i32", (4,)), synth.ColSpec("act", "i32", ())],
                  [synth.ColSpec("obs", "f32", (4,)), synth.ColSpec("action", "i32", ())]):
        Q = Pair(capacity=Cs * R, seq_len=3, colspecs=other, R=R, mirror=False)
        with pytest.raises(G.GearError, match="schema"):
            Q.t.load(path)
        Q.close()
    # truncated file: refused before anything is overwritten
    trunc = str(tmp_path / "trunc.gear")
    with open(trunc, "wb") as f:
        f.write(open(path, "rb").read()[:-100])
    key0, seq0, gen0 = P.t.read_state()
    with pytest.raises(G.GearError, match="bytes"):
        P.t.load(trunc)
    key1, seq1, gen1 = P.t.read_state()
    assert np.array_equal(key0, key1) and np.array_equal(seq0, seq1) and np.array_equal(gen0, gen1)
    P.check_state()
    torch.cuda.synchronize()
    P.close()
