"""A/B probe (not a test): the streamed host job (lbg_run_host) on the 512^3 config-2 block —
wall time per call for several slab sizes, first (allocating) and repeated calls — next to the
PCIe copy rates of the same bytes (H2D alone, D2H alone, both directions at once).

    python tests/ab_job.py [n] [steps]
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2303_11811_b200 import lbdem  # noqa: E402
from paper_2303_11811_b200 import lbg as abi  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    torch.cuda.set_device(0)
    lib = abi.load()
    dims = (n, n, n)
    blk = lbdem.Block(dims)
    blk.set_periodic_wrap((1, 1, 1))
    blk.init_shear_wave(dims)
    p = lbdem.FluidParams(0.8)
    nbytes = 8 * 19 * (n + 2) ** 3
    hp = C.c_void_p()
    lbdem.check(lib.lbg_host_alloc(nbytes, C.byref(hp)))
    host = np.ctypeslib.as_array(C.cast(hp, C.POINTER(C.c_double)), shape=(19, n + 2, n + 2, n + 2))
    lbdem.check(lib.lbg_download_src(blk.h, hp))
    cells = n ** 3

    # raw PCIe rates on the same pinned buffer (torch copies, separate streams)
    hb = torch.from_numpy(host.reshape(-1)[: nbytes // 8 // 2 * 2])
    half = hb.numel() // 2
    d1 = torch.empty(half, dtype=torch.float64, device="cuda")
    d2 = torch.empty(half, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for name, fn in [
        ("h2d", lambda: d1.copy_(hb[:half], non_blocking=True)),
        ("d2h", lambda: hb[:half].copy_(d1, non_blocking=True)),
    ]:
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps({"copy": name, "GB": round(half * 8 / 1e9, 2), "GBps": round(half * 8 / dt / 1e9, 1)}))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d1.copy_(hb[:half], non_blocking=True)
    with torch.cuda.stream(s2):
        hb[half:2 * half].copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"copy": "both directions", "GB_each": round(half * 8 / 1e9, 2),
                      "GBps_each": round(half * 8 / dt / 1e9, 1)}))
    del d1, d2
    torch.cuda.empty_cache()

    for slab in [int(x) for x in os.environ.get("AB_SLABS", "16,8,32,4").split(",")]:
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            blk.run_host(p, host, steps, slab)
            dt = time.perf_counter() - t0
            print(json.dumps({"slab": slab, "rep": rep, "steps": steps, "s": round(dt, 4),
                              "mlups": round(cells * steps / dt / 1e6, 1)}))
    lib.lbg_host_free(hp)
    blk.close()


if __name__ == "__main__":
    main()
