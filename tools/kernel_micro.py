"""Latency / bandwidth of the selection kernels (development tool).

For a table of N trajectories (one 16-byte column so the fill is cheap) and
batch B: the time of gear_sample on a dirty table (K1 scan + K2 sample), on a
clean table (K2 only), and of gear_update_priorities (K6), each the median of
50 calls timed with CUDA events on the calling stream.  The scan's HBM
fraction uses 16 B per key (read key, write cdf) over MEASURED_PEAKS hbm_gbs.
One JSON line per (N, B, strategy)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2310_05205_b200 as gear  # noqa: E402


def med_us(fn, stream, reps=50):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        stream.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6650.0
    stream = torch.cuda.Stream()
    for N in (100_000, 1_000_000, 10_000_000):
        t = gear.Table(N, 1, [gear.Column("x", gear.GEAR_U8, (16,))], None, max_batch=4096)
        rows = torch.zeros((1 << 20, 16), dtype=torch.uint8, device="cuda")
        prio = synth.priorities(N, seed=1, zero_frac=0.01)
        for k0 in range(0, N, 1 << 20):
            m = min(1 << 20, N - k0)
            gear.gear_insert(t.handle, 0, m, [rows], prio[k0:k0 + m], None, stream)
        stream.synchronize()
        for B in (512, 4096):
            idx = torch.empty(B, dtype=torch.int64, device="cuda")
            w = torch.empty(B, dtype=torch.float32, device="cuda")
            p = torch.from_numpy(synth.priorities(B, seed=7)).cuda()
            for strat in ("prioritized", "uniform"):
                sc = gear.STRATEGIES[strat]
                seed = [0]

                def sample():
                    seed[0] += 1
                    gear.gear_sample(t.handle, sc, B, seed[0], 0.4, idx, w, None, None, stream)

                def dirty_sample():
                    gear.gear_update_priorities(t.handle, 1, idx, p, gear.GEAR_F64, None, stream)
                    sample()

                def update():
                    gear.gear_update_priorities(t.handle, B, idx, p, gear.GEAR_F64, None, stream)

                sample()
                t_clean = med_us(sample, stream)
                t_upd1 = med_us(lambda: gear.gear_update_priorities(t.handle, 1, idx, p, gear.GEAR_F64,
                                                                    None, stream), stream)
                t_dirty = med_us(dirty_sample, stream) - t_upd1
                t_upd = med_us(update, stream)
                scan_us = max(t_dirty - t_clean, 1e-3)
                print(json.dumps({"N": N, "B": B, "strategy": strat, "sample_clean_us": round(t_clean, 2),
                                  "sample_dirty_us": round(t_dirty, 2), "scan_us": round(scan_us, 2),
                                  "scan_hbm_frac": round(16 * N / (scan_us * 1e-6) / 1e9 / peak, 3),
                                  "update_us": round(t_upd, 2)}), flush=True)
        err, _ = t.sync()
        assert err == 0
        t.close()


if __name__ == "__main__":
    main()
