"""A/B of the coupled sweep on config 5's dilute bed (bench.coupled_sweep_roofline with
bench.CONFIG5_1GPU: 12,500 spheres in one 512^3 block): one JSON line per run, kernel variants
chosen by the LBG_* environment switches."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

r = bench.coupled_sweep_roofline(steps=int(os.environ.get("AB_STEPS", "10")), cfg=bench.CONFIG5_1GPU, n=512,
                                 label="config 5 bed, one 512^3 block")
env = {k: v for k, v in os.environ.items() if k.startswith("LBG_")}
print(json.dumps({"env": env, "sweep_ms": r["sweep_ms"], "frac": r["roofline"]["frac"],
                  "one_entry": r["one_entry_cells"], "two_entry": r["two_entry_cells"]}))
