"""CUDA-graph replay of the hot path (W = 1): a sample -> collect -> update
step is captured once and replayed; the device-resident seed counter and
update epoch advance on the device, so every replay must equal the oracle's
next step (draw key = seed0 + i)."""
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


@pytest.mark.parametrize("R", [1, 3])
def test_graph_replayed_steps_match_oracle(torch_cuda, R):
    import oracle
    import paper_2310_05205_b200 as G
    from gpu_harness import Pair
    torch = torch_cuda
    cfg = synth.CONFIGS["c1"]
    N = 1023 if R == 3 else cfg.capacity
    P = Pair(capacity=N, seq_len=cfg.seq_len, colspecs=cfg.cols, R=R)
    P.fill(synth.priorities(N, seed=4, zero_frac=0.1))
    B, beta, seed0 = 64, 0.4, 0x5EED0000
    h = P.t.handle
    G.gear_table_set_tuning(h, "device_seed", seed0)
    idx = torch.empty(B, dtype=torch.int64, device="cuda")
    w = torch.empty(B, dtype=torch.float32, device="cuda")
    outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in P.rb]
    pools = [synth.priorities(B, seed=100 + k, zero_frac=0.05) for k in range(2)]
    dpools = [torch.from_numpy(p).cuda() for p in pools]
    strat = G.GEAR_PRIORITIZED | G.GEAR_SAMPLE_DEVICE_SEED

    def step(k):
        G.gear_sample(h, strat, B, 0, beta, idx, w)
        G.gear_collect(h, B, idx, list(range(len(outs))), outs)
        G.gear_update_priorities(h, B, idx, dpools[k], G.GEAR_F64)

    # eager step 0 (also warms up), then capture steps 1 and 2 as one graph
    step(0)
    torch.cuda.synchronize()
    seeds = [seed0]
    graph = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s, capture_error_mode="thread_local"):
            step(1)
    torch.cuda.synchronize()
    # capture does not execute: the counter is still seed0 + 1
    results = []
    for rep in range(5):
        graph.replay()
        torch.cuda.synchronize()
        results.append((idx.cpu().numpy().view(np.uint64).copy(), w.cpu().numpy().copy(),
                        [o.cpu().numpy().copy() for o in outs]))
    err, _ = P.t.sync()
    assert err == 0
    # oracle: step 0 eager (seed0, pool 0), then 5 replays of step(1) (pool 1)
    st, oi, ow, _ = P.o.sample(oracle.PRIORITIZED, 1, 0, B, seed0, beta)
    P.o.update(oi, pools[0])
    for rep in range(5):
        st, oi, ow, _ = P.o.sample(oracle.PRIORITIZED, 1, 0, B, seed0 + 1 + rep, beta)
        gi, gw, gouts = results[rep]
        assert np.array_equal(gi, oi), f"replay {rep}: ids differ"
        np.testing.assert_allclose(gw, ow, rtol=1e-6)
        for c in range(len(gouts)):
            assert np.array_equal(gouts[c], oracle.collect(P.mirror[c], oi))
        P.o.update(oi, pools[1])
    key, _, _ = P.t.read_state()
    assert np.array_equal(key, P.o.key)
    P.close()
