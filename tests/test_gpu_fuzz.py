"""Randomised operation sequences against the oracle: inserts (host and device
priorities), allocate -> in-place rows -> commit, priority updates (fused and
grid-wide, with generations and stale entries), samples of every strategy,
collects, CDF layout switches and a checkpoint
round trip in the middle -- the state and every result compared after every
operation."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
G = __import__("paper_2310_05205_b200")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


@pytest.mark.parametrize("seed,removal,alpha", [(1, 0, 1.0), (2, 1, 0.7), (3, 0, 0.6), (4, 1, 1.0),
                                                (5, 0, 2.0), (6, 1, 0.5)])
def test_random_operation_sequences(torch_cuda, tmp_path, seed, removal, alpha):
    import oracle
    from gpu_harness import Pair
    cols = [synth.ColSpec("obs", "f32", (6,)), synth.ColSpec("act", "u8", (3,))]
    R, Cs = 3, 300
    P = Pair(capacity=Cs * R, seq_len=2, colspecs=cols, R=R, removal=removal, alpha=alpha)
    rng = np.random.default_rng(seed)
    strategies = [G.GEAR_UNIFORM, G.GEAR_WEIGHTED, G.GEAR_PRIORITIZED, G.GEAR_FIFO, G.GEAR_LIFO,
                  G.GEAR_TOPK]
    saved = False
    for step in range(300):
        op = int(rng.integers(0, 8))
        s = int(rng.integers(0, R))
        if op == 0:                                     # insert, host priorities
            P.insert(s, synth.priorities(int(rng.integers(1, 200)), seed=step, zero_frac=0.1))
        elif op == 1:                                   # insert, device rows
            P.insert(s, synth.priorities(int(rng.integers(1, 120)), seed=step), device_src=True)
        elif op == 2:                                   # allocate -> rows -> commit
            ids = P.allocate(s, int(rng.integers(1, 40)))
            if ids is not None:
                P.write_rows(ids)
                keep = ids[rng.random(ids.size) < 0.8]  # some stay ongoing for a while
                if keep.size:
                    P.commit(s, keep, synth.priorities(keep.size, seed=step))
        elif op == 3:                                   # commit whatever is still ongoing
            o = P.o
            lo, hi = s * Cs, (s + 1) * Cs
            ongoing = [g for g in range(lo, hi) if o.gen[g] > 0 and o.seq[g] == 0]
            if ongoing:
                P.commit(s, np.array(ongoing, np.uint64), synth.priorities(len(ongoing), seed=step))
        elif op == 4:                                   # priority update with stale entries
            G.gear_table_set_tuning(P.t.handle, "update_fused", int(rng.integers(0, 2)))
            ids = rng.integers(0, Cs * R, int(rng.integers(1, 300))).astype(np.uint64)
            gen = P.o.gen[ids.astype(np.int64)].copy()
            gen[rng.random(ids.size) < 0.1] += 1
            P.update(ids, rng.lognormal(0, 2, ids.size) * (rng.random(ids.size) > 0.1), gen=gen)
        elif op == 5:                                   # sample + collect
            strat = strategies[int(rng.integers(0, len(strategies)))]
            B = int(rng.integers(1, 200))
            idx = P.check_sample(strat, B, 1000 + step, beta=float(rng.random()))
            if idx is not None:
                P.check_collect(idx)
        elif op == 6:                                   # CDF layout switch
            G.gear_table_set_tuning(P.t.handle, "cdf_levels", int(rng.integers(1, 3)))
        elif op == 7 and not saved and step > 40:       # checkpoint round trip
            path = str(tmp_path / f"fuzz_{seed}.gear")
            ongoing = [(g // Cs, g) for g in range(Cs * R) if P.o.gen[g] > 0 and P.o.seq[g] == 0]
            if ongoing:                                 # an in-flight allocation: refused
                with pytest.raises(G.GearError) as e:
                    P.t.save(path)
                assert e.value.status == G.GEAR_ERR_STATE
                for sh in range(R):
                    ids = np.array([g for q, g in ongoing if q == sh], np.uint64)
                    if ids.size:
                        P.commit(sh, ids, synth.priorities(ids.size, seed=step + sh))
            P.t.save(path)
            Q = Pair(capacity=Cs * R, seq_len=2, colspecs=cols, R=R, removal=removal, alpha=alpha,
                     mirror=False)
            Q.t.load(path)
            Q.o, Q.mirror, Q.content, Q.next_traj = P.o, P.mirror, P.content, P.next_traj
            P.t.close()
            P = Q
            saved = True
        P.check_state()
    for strat in strategies:
        idx = P.check_sample(strat, 64, 7)
        if idx is not None:
            P.check_collect(idx)
    assert oracle.OK == 0
    P.close()
