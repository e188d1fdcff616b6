"""Collect-kernel sweep on a bench-shaped table (development tool).
Times gear_collect alone with CUDA events for LSU and TMA variants
(ctas per SM x stages x stage bytes), 3 interleaved rounds of 20 launches;
prints one JSON line per variant (median / min over the 60 launches)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402

VARIANTS = [("lsu", 0, 0, 0), ("tma", 1, 6, 32768), ("tma", 1, 8, 16384), ("tma", 2, 3, 16384),
            ("tma", 2, 4, 16384), ("tma", 2, 6, 16384), ("tma", 2, 3, 32768), ("tma", 3, 4, 16384),
            ("tma", 4, 3, 16384), ("tma", 4, 2, 16384), ("tma", 2, 2, 32768), ("tma", 3, 2, 32768),
            ("tma", 4, 4, 8192), ("tma", 6, 4, 8192)]


def tune(h, impl, ctas, stages, chunk):
    S = gear.gear_table_set_tuning
    S(h, "collect_impl", 1 if impl == "tma" else 0)
    if impl == "tma":
        S(h, "tma_ctas_per_sm", 1)
        S(h, "tma_stages", 2)
        S(h, "tma_chunk", chunk)
        S(h, "tma_ctas_per_sm", ctas)
        S(h, "tma_stages", stages)


def main():
    cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cap = int(sys.argv[2]) if len(sys.argv) > 2 else 30000
    cfg = synth.CONFIGS[cfg_name]
    stream = torch.cuda.Stream()
    t, _ = bench.build_table(cfg, None, 1, 0, cap, stream)
    B = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.batch
    idx = torch.empty(B, dtype=torch.int64, device="cuda")
    outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
    payload = B * sum(t.row_bytes)
    times = {v: [] for v in VARIANTS}
    it = 0
    for rnd in range(3):
        for v in VARIANTS:
            tune(t.handle, *v)
            for i in range(23):
                it += 1
                gear.gear_sample(t.handle, gear.STRATEGIES[cfg.strategy], B, 1000 + it, 0.4, idx,
                                 None, None, None, stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                gear.gear_collect(t.handle, B, idx, list(range(len(outs))), outs, stream)
                e1.record(stream)
                stream.synchronize()
                if i >= 3:
                    times[v].append(e0.elapsed_time(e1))
    for v, ts in times.items():
        ts.sort()
        med = ts[len(ts) // 2]
        print(json.dumps({"config": cfg_name, "capacity": cap, "B": B, "impl": v[0], "ctas": v[1],
                          "stages": v[2], "chunk": v[3], "median_us": round(med * 1e3, 2),
                          "min_us": round(ts[0] * 1e3, 2), "payload_GBps": round(payload / med / 1e6, 1),
                          "rw_GBps": round(2 * payload / med / 1e6, 1)}), flush=True)
    err, _ = t.sync()
    assert err == 0
    t.close()


if __name__ == "__main__":
    main()
