"""A/B of the K3 mapping on config 3's bed (10^4 spheres in one 256^3 block): maps the bed
AB_MAPS times and prints the mean wall time of Block.map (zero fill, binning, mapping kernel,
segment lists; run under `ncu --metrics gpu__time_duration.sum` for per-kernel times) and a
hash of the fraction field, so variants selected by LBG_* switches can be compared bitwise."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "integration"))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import dropin  # noqa: E402
from paper_2303_11811_b200 import lbdem  # noqa: E402

n = 256
sim = dropin.DropinSim(bench.config3(), (n, n, n))
rows = sim.particles()
sim.close()
r = 5.0
snaps = {"id": rows[:, 0].astype(np.int32), "x": rows[:, 1:4].copy(), "r": np.full(len(rows), r),
         "f_r": np.full(len(rows), lbdem.f_of_r(r)), "u": rows[:, 4:7].copy(), "w": rows[:, 7:10].copy()}
blk = lbdem.Block((n, n, n), coupling=True)
reps = int(os.environ.get("AB_MAPS", "10"))
blk.map(snaps)
blk.sync()
t0 = time.perf_counter()
for _ in range(reps):
    blk.map(snaps)
blk.sync()
dt = (time.perf_counter() - t0) / reps
fr = blk.download_fraction()
h = hashlib.sha256()
c = fr["count"]
h.update(c.tobytes())
h.update(fr["btot"].tobytes())
for k, lo in (("id0", 1), ("b0", 1), ("id1", 2), ("b1", 2)):  # entries only (the rest is stale)
    h.update(np.ascontiguousarray(fr[k][c >= lo]).tobytes())
env = {k: v for k, v in os.environ.items() if k.startswith("LBG_")}
print(json.dumps({"env": env, "map_ms": round(dt * 1e3, 4), "fraction_sha": h.hexdigest()[:16],
                  "covered": int((fr["count"] > 0).sum())}))
blk.close()
