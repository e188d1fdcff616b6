"""C-ABI argument errors (include/gear.h): every entry point rejects bad
arguments with the documented status and leaves the table usable."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = __import__("paper_2310_05205_b200")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    return torch


def _raises(status, fn, *a, **kw):
    with pytest.raises(G.GearError) as e:
        fn(*a, **kw)
    assert e.value.status == status, (e.value.status, status)


def test_invalid_arguments(torch_cuda):
    torch = torch_cuda
    col = [G.Column("x", G.GEAR_U8, (4,))]
    INV = G.GEAR_ERR_INVALID_ARG
    _raises(INV, G.Table, 1001, 1, col, None, shards_per_rank=2)      # N % S != 0
    _raises(INV, G.Table, 64, 0, col, None)                          # seq_len 0
    _raises(INV, G.Table, 64, 1, col, None, alpha=-1.0)              # alpha < 0
    _raises(INV, G.Table, 64, 1, col, None, alpha=float("nan"))
    _raises(INV, G.Table, 64, 1, col, None, frac_bits=63)
    t = G.Table(128, 1, col, None, shards_per_rank=2, max_batch=64)
    h = t.handle
    rows = [torch.zeros((4, 4), dtype=torch.uint8, device="cuda")]
    idx = torch.zeros(8, dtype=torch.int64, device="cuda")
    _raises(INV, t.insert, 2, rows, np.ones(4))                      # shard not owned
    _raises(G.GEAR_ERR_BAD_PRIORITY, t.insert, 0, rows, np.array([1.0, -1.0, 1.0, 1.0]))
    t.insert(0, rows, np.ones(4))
    _raises(INV, G.gear_update_priorities, h, 65, torch.zeros(65, dtype=torch.int64, device="cuda"),
            torch.ones(65, dtype=torch.float64, device="cuda"), G.GEAR_F64)   # n > max_batch
    _raises(INV, G.gear_update_priorities, h, 8, idx, torch.ones(8, device="cuda"), G.GEAR_I32)
    _raises(INV, G.gear_sample, h, 9, 8, 1, 0.4, idx)                # bad strategy
    _raises(INV, G.gear_sample, h, G.GEAR_UNIFORM, 65, 1, 0.4,
            torch.zeros(65, dtype=torch.int64, device="cuda"))       # B > max_batch
    _raises(INV, G.gear_sample, h, G.GEAR_PRIORITIZED, 8, 1, float("inf"), idx)
    out = [torch.empty((8, 4), dtype=torch.uint8, device="cuda")]
    _raises(INV, G.gear_collect, h, 8, idx, [3], out)                # bad column
    _raises(INV, G.gear_table_set_tuning, h, "no_such_knob", 1)
    _raises(INV, G.gear_table_set_tuning, h, "cdf_levels", 3)
    _raises(INV, G.gear_table_set_tuning, h, "tma_stages", 5)
    _raises(INV, G.gear_allocate, h, 5, 4, idx)                      # shard out of range
    _raises(INV, G.gear_allocate, h, 0, 65, torch.zeros(65, dtype=torch.int64, device="cuda"))
    _raises(INV, G.gear_commit, h, 3, 4, idx, np.ones(4))
    _raises(INV, G.gear_column_id, h, "nope")
    _raises(G.GEAR_ERR_STATE, G.gear_read_cdf, h)                    # no CDF built yet
    _raises(INV, G.gear_sample, h, G.GEAR_UNIFORM, 8, 1, 0.4, idx, flags=0x4)   # unknown flag
    _raises(INV, G.gear_table_set_tuning, h, "collect_dynamic", 2)
    _raises(INV, G.gear_table_set_tuning, h, "collect_evict_first", -2)
    # the table still works after the rejected calls
    t.sample(G.GEAR_UNIFORM, 8, 1, 0.0, idx)
    t.collect(idx, [0], out)
    torch.cuda.synchronize()
    err, _ = t.sync()
    assert err == 0
    assert set(idx.cpu().numpy().tolist()) <= {0, 1, 2, 3}
    t.close()
