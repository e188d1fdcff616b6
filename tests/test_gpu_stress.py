"""Stress test of the lock-free device protocols (compute-sanitizer is closed
on this GPU pool: profiles/r02a/compute_sanitizer_refused.log).  Thousands of
CUDA-graph-replayed steps -- sample (device seed counter) -> collect ->
collective-form priority update -- over randomised table shapes, batch
sizes, CDF layouts and strategies, every step compared with the oracle.

What it exercises (each is device-resident state advanced by the kernels
and re-armed by the last CTA of a launch, so a replay that skips a re-arm or
races on a counter shows up as a wrong id / weight / row / key):
  * the decoupled look-back scan's tickets, epoch-alternated status words,
    exit counter and CDF parity (cdf_levels 1) and the two-level scan's
    per-shard arrival counters, dirty bits and buffer modes (cdf_levels 2);
  * the sample kernel's last-block q_min slot and done counter (IS weights),
    and the device seed counter;
  * the update kernel's 40-bit tag epoch (last writer wins, duplicates);
  * TopK's radix-select histograms and counters; FIFO/LIFO ring walks;
  * the collect engine's persistent TMA ring (mbarrier phases).
"""
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


CASES = [  # (R, Cs, B, cdf_levels, strategy, steps per graph, replays, scan_chunk)
    (1, 4096, 64, 1, "prioritized", 10, 60, 0),
    (3, 1500, 37, 2, "prioritized", 10, 60, -1),
    (8, 700, 1000, 1, "weighted", 5, 60, 1),
    (5, 9000, 512, 2, "uniform", 10, 40, -1),
    (2, 20000, 256, 1, "prioritized", 8, 40, 0),
    (2, 20000, 256, 1, "prioritized", 8, 40, 3),
    (3, 50000, 512, 1, "uniform", 8, 40, 1),
    (4, 3000, 128, 2, "topk", 10, 40, -1),
    (2, 2500, 96, 1, "fifo", 5, 40, -1),
    (1, 30000, 4096, 2, "prioritized", 4, 40, -1),
]


@pytest.mark.parametrize("case", CASES, ids=[f"R{c[0]}-Cs{c[1]}-B{c[2]}-L{c[3]}-{c[4]}-K{c[7]}" for c in CASES])
def test_graph_replay_stress(torch_cuda, case):
    import oracle
    import paper_2310_05205_b200 as G
    from gpu_harness import ORACLE_STRATEGY, Pair
    torch = torch_cuda
    R, Cs, B, levels, sname, S, reps, chunk = case
    cols = [synth.ColSpec("obs", "f32", (3,)), synth.ColSpec("tok", "u8", (5,))]
    N = R * Cs
    P = Pair(capacity=N, seq_len=2, colspecs=cols, R=R, max_batch=max(4096, B))
    P.fill(synth.priorities(N, seed=R * 7 + B, zero_frac=0.05))
    h = P.t.handle
    G.gear_table_set_tuning(h, "cdf_levels", levels)
    G.gear_table_set_tuning(h, "scan_chunk", chunk)
    strat = G.STRATEGIES[sname]
    ostrat = ORACLE_STRATEGY[strat]
    seed0, beta = 0x5EED1000 + B, 0.4
    G.gear_table_set_tuning(h, "device_seed", seed0)
    rng = np.random.default_rng(B + R)
    idx = [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(S)]
    w = [torch.empty(B, dtype=torch.float32, device="cuda") for _ in range(S)]
    outs = [[torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in P.rb] for _ in range(S)]
    # step i of the graph updates the sampled ids with pool[i] (duplicates and
    # zeros included: last writer wins, zero keys leave the CDF)
    pools = [rng.lognormal(0, 1.5, B) * (rng.random(B) > 0.05) for _ in range(S)]
    dpools = [torch.from_numpy(p).cuda() for p in pools]
    upd = sname != "fifo"          # FIFO order does not depend on the keys' values

    def step(i):
        G.gear_sample(h, strat, B, 0, beta, idx[i], w[i], flags=G.GEAR_SAMPLE_DEVICE_SEED)
        G.gear_collect(h, B, idx[i], list(range(len(P.rb))), outs[i])
        if upd:
            G.gear_update_priorities(h, B, idx[i], dpools[i], G.GEAR_F64)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s, capture_error_mode="thread_local"):
            for i in range(S):
                step(i)
    torch.cuda.synchronize()
    seed = seed0
    for rep in range(reps):
        graph.replay()
        torch.cuda.synchronize()
        for i in range(S):
            st, oi, ow, _ = P.o.sample(ostrat, 1, 0, B, seed, beta)
            seed += 1
            assert st == 0
            gi = idx[i].cpu().numpy().view(np.uint64)
            if not np.array_equal(gi, oi):
                raise AssertionError(f"replay {rep} step {i}: ids differ at {np.nonzero(gi != oi)[0][:8]}")
            np.testing.assert_allclose(w[i].cpu().numpy(), ow, rtol=1e-6, atol=0)
            for c in range(len(P.rb)):
                assert np.array_equal(outs[i][c].cpu().numpy(), oracle.collect(P.mirror[c], oi)), \
                    f"replay {rep} step {i} column {c}"
            if upd:
                P.o.update(oi, pools[i])
    err, _ = P.t.sync()
    assert err == 0, err
    P.check_state()
    P.close()
