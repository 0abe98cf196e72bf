"""A/B diagnostics of config 2's side records (bench.coupled_b0_roofline, bench.aa_roofline):
one JSON line each (kernel variants chosen by the LBG_* environment switches)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

env = {k: v for k, v in os.environ.items() if k.startswith("LBG_")}
b0 = bench.coupled_b0_roofline()
aa = bench.aa_roofline()
print(json.dumps({"env": env, "b0_ms": b0["sweep_ms"], "b0_frac": b0["roofline"]["frac"],
                  "aa_ms": aa["sweep_ms"], "aa_frac": aa["roofline"]["frac"], "aa_bytes": aa["device_bytes"]}))
