"""A/B probe (not a test): config 3's coupled step through the drop-in and on the reference for
several block decompositions / worker counts (bench.coupled_step, best of 3).

    AB_BLOCKS="2,2,2:8;4,2,2:16" python tests/ab_blocks.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

for spec in os.environ.get("AB_BLOCKS", "2,2,2:8;4,2,2:16").split(";"):
    b, w = spec.split(":")
    blocks = tuple(int(v) for v in b.split(","))
    r = bench.coupled_step(4, os.environ.get("AB_REF", "1") == "1", ref_steps=1, blocks=blocks, workers=int(w))
    r.pop("workload", None)
    print(json.dumps(r), flush=True)
