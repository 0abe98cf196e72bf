#!/usr/bin/env python
"""Config 5 (BASELINE.json): fluidized-bed four-way coupled PSM + DEM, weak and strong
scaling over the GPUs of one box, through the drop-in build (the reference Simulation with
its GPU-side operators on liblbg; host DEM = the reference's code).

    python bench_config5.py --gpus N [--steps K] [--edge 512] [--per-gpu 12500]
    python bench_config5.py --gpus N --mode strong [--steps K]

Weak scaling as SURVEY §8(d): domain (edge*N) x edge x edge, block grid {N,1,1} (x-slabs, so
the bottom-settled bed splits evenly), edge^3 cells and `per_gpu` spheres (d = 10) per GPU.
Strong scaling: the fixed 1024 x 512 x 512 bed (2.7e8 cells, 10^5 spheres; about 120 GB on a
single GPU) split into {N,1,1} x-slabs. Either way `--blocks-per-gpu` consecutive x-slab blocks
per GPU (LBDEM_GPU_SPREAD=1), one reference worker thread per block, no host PDF mirror
(LBDEM_GPU_HOST_MIRROR=0), the pushed halo between blocks (LBDEM_GPU_HALO, default push).
Prints one JSON line with, per force mode (scratch = bitwise PARITY partials, fused), the
reference's own per-category TimingReport (perf.hpp:17-51) and MLUPS = cells * steps / wall time.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "integration"))

CATS = ("PSM", "PSM-comm", "mapping", "setU", "redF", "PD", "PD-comm", "other")
CFG = ('{{"scenario":"fluidized_bed_dense","domain":[{nx},{n},{n}],"blocks":[{g},1,1],'
       '"workers":{g},"particles":{{"count":{p}}},"physical":{{"diameter_cells":10}},'
       '"fluid":{{"bc":{{"xm":"no_slip","xp":"no_slip","ym":"no_slip","yp":"no_slip",'
       '"zm":"velocity","zp":"pressure"}}}},'
       '"dem":{{"k_n":230,"d_n":520,"k_t":65,"d_t":260,"subcycles":10,"settle_subcycles":{settle}}}}}')


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--edge", type=int, default=512)
    ap.add_argument("--per-gpu", type=int, default=12500)
    ap.add_argument("--settle", type=int, default=100)
    ap.add_argument("--force", choices=["scratch", "fused", "both"], default="both",
                    help="scratch: reference semantics, bitwise PARITY partials; fused: per-particle sums "
                         "inside the PSM kernel (tolerance); both: one run each, scratch first")
    ap.add_argument("--mode", choices=["weak", "strong"], default="weak")
    ap.add_argument("--blocks-per-gpu", type=int, default=0,
                    help="x-slab blocks per GPU (consecutive ids), one host worker each: spreads the host DEM "
                         "(0: weak up to 8 within the host CPUs; strong one worker per host CPU, the largest power of two <= CPUs / GPUs, "
                         "at most 16 per GPU — profiles/r02_c5blocks*.log)")
    args = ap.parse_args()
    if args.blocks_per_gpu <= 0:
        if args.mode == "strong":
            per = max(1, (os.cpu_count() or 4) // args.gpus)
            bpg = 1
            # (at most 16 per GPU: 32 slabs of the 1024 x 512 x 512 bed did not fit one GPU)
            while 2 * bpg <= per and 2 * bpg <= 16:
                bpg *= 2
            args.blocks_per_gpu = bpg
        else:
            # weak: up to 8 x-slab blocks per GPU within the host's CPUs (1 GPU: 23-31 ms per
            # step with 8 vs 33 with 4 and 28-34 with 16, whose thin slabs cost more sweep —
            # profiles/r02_c5weak_ab.log)
            per = max(1, (os.cpu_count() or 4) // args.gpus)
            bpg = 1
            while 2 * bpg <= min(8, per):
                bpg *= 2
            args.blocks_per_gpu = bpg
    os.environ["LBDEM_GPU_SPREAD"] = "1"
    os.environ["LBDEM_GPU_HOST_MIRROR"] = "0"
    os.environ["LBDEM_GPU_BLOCKS_PER_DEVICE"] = str(args.blocks_per_gpu)
    import torch  # noqa: F401  (CUDA plumbing)
    import dropin
    g, n = args.gpus, args.edge
    if args.mode == "strong":
        nx, particles = 2 * n, 100000
    else:
        nx, particles = n * g, args.per_gpu * g
    nb = g * args.blocks_per_gpu
    cfg = CFG.format(nx=nx, n=n, g=nb, p=particles, settle=args.settle)
    cells = nx * n * n
    out = {"workload": f"config 5 {args.mode}: {nx}x{n}x{n} fluidized bed, {particles} spheres d=10, "
                       f"blocks {{{nb},1,1}}, {args.blocks_per_gpu} per GPU (one host worker each), "
                       f"host DEM (reference)",
           "blocks_per_gpu": args.blocks_per_gpu, "scaling": args.mode, "n_gpus": g, "steps": args.steps,
           "particles": particles, "halo": os.environ.get("LBDEM_GPU_HALO", "push")}
    for mode in (("scratch", "fused") if args.force == "both" else (args.force,)):
        os.environ["LBDEM_GPU_FORCE"] = mode
        t0 = time.perf_counter()
        sim = dropin.DropinSim(cfg, (nx, n, n))
        setup = time.perf_counter() - t0
        sim.run(1)
        sim.reset_timers()
        t0 = time.perf_counter()
        sim.run(args.steps)
        dt = time.perf_counter() - t0
        cat = sim.timings()
        out[mode] = {
            "force_mode": mode, "ms_per_step": round(dt * 1e3 / args.steps, 2),
            "mlups": round(cells * args.steps / dt / 1e6, 1),
            "mlups_per_gpu": round(cells * args.steps / dt / 1e6 / g, 1),
            "categories_ms_per_step": {c: round(v * 1e3 / args.steps, 3) for c, v in zip(CATS, cat)},
            "setup_s": round(setup, 1)}
        sim.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
