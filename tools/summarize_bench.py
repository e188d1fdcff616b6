"""One line per bench JSON of a suite directory."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] + "/bench_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(f.split("/")[-1], "unparsable:", e)
        continue
    if d.get("impl") == "reference":
        print(f.split("/")[-1], "reference %.4g %s" % (d["value"], d["unit"]), d["cpu_baseline"]["sample"][:80])
        continue
    r = d["roofline"]
    cb = d.get("cpu_baseline", {})
    print(f.split("/")[-1], "%.3fM traj/s" % (d["value"] / 1e6), "ms %.4f" % d["ms_per_step"],
          "e2e %.3fM" % (d["e2e"]["value"] / 1e6), r["bound"], "frac %.3f" % r["frac"],
          "step_frac %.3f" % r.get("step_frac", 0), "peak %.1f" % r["peak"],
          "sel_only %.4f" % d.get("selection", {}).get("only_ms_per_step", 0),
          "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"),
          "cpu %.4g" % cb.get("value", 0), "launches", d.get("gpu_launches"))
