"""bench.py's reference arm runs on the CPU (the oracle, as it stands): its
JSON line carries the contract's keys, and under a multi-rank launch only rank
0 prints (tests need no GPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env):
    env = dict(os.environ, **extra_env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "c1", "--steps", "2", "--warmup", "3", "--cpu-budget", "0.5"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.strip()]


def test_reference_arm_json_line():
    lines = _run({"RANK": "0", "WORLD_SIZE": "1"})
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "trajectories/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "c1_tiny"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] == 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_print_nothing():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}) == []


def test_auto_assignment_by_placement():
    """--assign auto: owner-affine for tables with HBM columns (c1, c2, c4),
    contiguous slices for all-host tables (c3, c5); explicit choices stay."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    for cfg, want in (("c1", "owner"), ("c2", "owner"), ("c3", "contiguous"), ("c4", "owner"),
                      ("c5", "contiguous")):
        a = argparse.Namespace(config=cfg, strategy=None, assign="auto")
        assert bench.resolve_assign(a) == want, cfg
    a = argparse.Namespace(config="c3", strategy=None, assign="owner")
    assert bench.resolve_assign(a) == "owner"
