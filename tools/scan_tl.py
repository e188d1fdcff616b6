"""Per-CTA timeline of one full CDF rebuild (A/B build with -DGEAR_SCAN_TL):
python tools/scan_tl.py N  (GEAR_LIB=paper_2310_05205_b200/ab/libgear_tl.so).
Each variant is rebuilt 3 times; the kernel's device printf lines of the last
rebuild (every 8th CTA: entry, phase marks, exit in %globaltimer ns) are
summarised: launch span, CTA start skew, phase durations, exit spread."""
import os
import subprocess
import sys

if len(sys.argv) > 2 and sys.argv[2] == "--child":
    import numpy as np
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth
    import paper_2310_05205_b200 as gear
    N = int(sys.argv[1])
    t = gear.Table(N, 1, [gear.Column("x", gear.GEAR_U8, (16,))], None, max_batch=4096)
    s = torch.cuda.Stream()
    rows = torch.zeros((1 << 20, 16), dtype=torch.uint8, device="cuda")
    prio = synth.priorities(N, seed=1, zero_frac=0.01)
    for k0 in range(0, N, 1 << 20):
        m = min(1 << 20, N - k0)
        gear.gear_insert(t.handle, 0, m, [rows], prio[k0:k0 + m], None, s)
    idx = torch.zeros(1, dtype=torch.int64, device="cuda")
    p1 = torch.ones(1, dtype=torch.float64, device="cuda")
    for name, levels, chunk in [("tile", 1, 0), ("chunk", 1, 1), ("s2p", 2, -1)]:
        gear.gear_table_set_tuning(t.handle, "cdf_levels", levels)
        gear.gear_table_set_tuning(t.handle, "scan_chunk", chunk)
        for r in range(3):
            if levels == 1:
                gear.gear_update_priorities(t.handle, 1, idx, p1, gear.GEAR_F64, None, s)
            else:
                gear.gear_table_set_tuning(t.handle, "cdf_levels", 2)
            s.synchronize()
            print(f"MARK {name} {r}", flush=True)
            gear.gear_sample(t.handle, gear.GEAR_PRIORITIZED, 1, 5, 0.4, idx, None, None, None, s)
            s.synchronize()
            torch.cuda.synchronize()
    print("MARK end", flush=True)
    t.close()
    sys.exit(0)

N = sys.argv[1] if len(sys.argv) > 1 else "10000000"
out = subprocess.run([sys.executable, __file__, N, "--child"], capture_output=True, text=True)
print(out.stderr[-2000:], file=sys.stderr)
with open(os.environ.get("SCAN_TL_RAW", os.devnull), "w") as f:
    f.write(out.stdout)
groups, cur = {}, None
for line in out.stdout.splitlines():
    if line.startswith("MARK"):
        cur = tuple(line.split()[1:])
        groups[cur] = []
    elif line.startswith("TL") and cur is not None:
        f = line.split()
        # TL <kernel> cta <b> sm <s> <t0> <t1> <t2> <t_end>
        groups[cur].append((f[1], int(f[3]), int(f[6]), int(f[7]), int(f[8]), int(f[9])))
for key, rows in groups.items():
    if len(key) < 2 or key[1] != "2":
        continue
    for kname in sorted({r[0] for r in rows}):
        rs = [r for r in rows if r[0] == kname]
        t0 = min(r[2] for r in rs)
        starts = sorted(r[2] - t0 for r in rs)
        ends = sorted(r[5] - t0 for r in rs)
        ph1 = sorted(r[3] - r[2] for r in rs if r[3])
        ph2 = sorted(r[4] - r[3] for r in rs if r[4] and r[3])
        q = lambda v: [v[0], v[len(v) // 2], v[-1]] if v else []
        print(f"N={N} {key[0]:5s} {kname:5s} ctas={len(rs)} span_ns={max(ends)} start(min/med/max)={q(starts)} "
              f"end={q(ends)} mark1-start={q(ph1)} mark2-mark1={q(ph2)}")
