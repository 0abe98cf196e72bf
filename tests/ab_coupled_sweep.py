"""A/B diagnostics of the coupled sweep on config 3's bed (bench.coupled_sweep_roofline): one
JSON line per run; kernel variants are chosen by the LBG_* environment switches."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

r = bench.coupled_sweep_roofline(steps=int(os.environ.get("AB_STEPS", "20")))
env = {k: v for k, v in os.environ.items() if k.startswith("LBG_")}
rec = {"env": env, "sweep_ms": r["sweep_ms"], "bc_ms": r["bc_ms"], "frac": r["roofline"]["frac"]}
if os.environ.get("AB_REDUCE_MS"):
    rec["reduce_ms"] = os.environ["AB_REDUCE_MS"]
print(json.dumps(rec))
