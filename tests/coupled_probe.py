"""Per-step timing probe of the config-3 coupled step through the drop-in (diagnostics)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "integration"))
import bench  # noqa: E402
import dropin  # noqa: E402

blocks = os.environ.get("PROBE_BLOCKS")  # e.g. "2,2,2": the reference's own worker parallelism
cfg = bench.CONFIG3
if blocks:
    import json as _j
    c = _j.loads(cfg)
    c["blocks"] = [int(v) for v in blocks.split(",")]
    c["workers"] = int(os.environ.get("PROBE_WORKERS", "8"))
    cfg = _j.dumps(c)
for mode in sys.argv[1:] or ["scratch"]:
    os.environ["LBDEM_GPU_FORCE"] = mode
    for k in range(int(os.environ.get("PROBE_SIMS", "1"))):  # fresh simulations (new workers) in one process
        sim = dropin.DropinSim(cfg, (256, 256, 256))
        for s in range(int(os.environ.get("PROBE_STEPS", "6"))):
            sim.reset_timers()
            t0 = time.perf_counter()
            sim.run(1)
            dt = time.perf_counter() - t0
            print(json.dumps({"mode": mode, "sim": k, "step": s, "ms": round(dt * 1e3, 2),
                              "cats": [round(v * 1e3, 2) for v in sim.timings()]}), flush=True)
        sim.close()
