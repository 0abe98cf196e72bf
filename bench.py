#!/usr/bin/env python
"""Benchmark of the GPU fluid step (BASELINE.json configs 2 and 4).

One step = one D3Q19 SRT fluid time step over the GPU's 512^3 block (fp64), exactly the
fluid phases of Simulation::step (sim.cpp:689-703) with coupling off:
  N = 1: fused pull stream-collide (K1) with the periodic wrap in-kernel -> swap
  N > 1: z-slab of a 512 x 512 x 512N periodic domain per GPU; x/y wrapped in-kernel;
         halo pack + NCCL send/recv on the comm stream (K7) || inner sweep k in [1,n-1) ->
         unpack -> outer sweep (k = 0, n-1) -> swap     (weak scaling, config 4)
Inputs: the validation.cpp:46-63 shear wave at tau = 0.8, initialised on the device.

`value` is MLUPS over all GPUs (cells * steps / max-over-ranks device time). `roofline`
uses 304 algorithmic bytes per lattice update (19 f64 pulled + 19 stored) and the sweep's
CUDA-event time measured in the timed region. `e2e` is the same K steps run as a job through
the C-ABI with host buffers: the state uploaded from pinned host memory, every step closed by
the reference's per-operator error check (one D2H of the stability counters), the final state
downloaded. `coupled_step` times config 3 (10^4 spheres, host DEM) through the drop-in build.
`cpu_baseline` times the reference itself (oracle/_ref) on this host.

`--impl reference` runs the unmodified reference CPU path (Simulation::step via
oracle/_ref) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MLUPS per GPU and % of HBM roofline at 1/2/4/8 B200; coupled step time"
BYTES_PER_LUP = 304  # 19 f64 loads + 19 f64 stores


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["lbg", "reference"], default="lbg")
    ap.add_argument("--n", "--edge", dest="n", type=int, default=512,
                    help="cells per axis of each GPU's block (--edge under torchrun, whose parser takes --n)")
    ap.add_argument("--tau", type=float, default=0.8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-coupled", action="store_true", help="skip the config-3 coupled-step timing")
    ap.add_argument("--coupled-steps", type=int, default=4, help="coupled steps per repetition (best of 3)")
    ap.add_argument("--halo", choices=["p2p", "nccl"], default="p2p",
                    help="N > 1: outer sweep stores into the neighbours over NVLink (p2p) or NCCL halo")
    ap.add_argument("--cpu-steps", type=int, default=3,
                    help="timed reference steps of the cpu_baseline leg (full domain, ~2.5 s each at 512^3)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()  # nvidia-smi needs a moment: start timing once it samples
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.02)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------------- reference CPU path
REF_CFG = ('{{"scenario":"custom","domain":[{nx},{ny},{nz}],"kernels":"openmp",'
           '"fluid":{{"tau":{tau},"coupling":false}},"dem":{{"subcycles":1}}}}')


def reference_sample(n, tau, steps, warmup=1):
    """Simulation::step of the unmodified reference (oracle/_ref) on the SAME workload the GPU
    arm runs: one periodic n^3 block (512^3: two 19-plane PdfField buffers of 41.3 GB host RAM),
    shear-wave init, coupling off, OpenMP on all host cores (perf.cpp:68-71 MLUPS). The host
    must hold the field: the run fails loudly rather than shrink the domain.
    Returns (MLUPS, sample description, threads, per-step seconds)."""
    from oracle.pyoracle import RefLib
    need = 2 * 19 * 8 * (n + 2) ** 3
    avail = host_mem_available()
    if avail is not None and need > 0.9 * avail:
        raise MemoryError(f"reference {n}^3 PdfField needs {need / 1e9:.1f} GB host RAM, "
                          f"MemAvailable is {avail / 1e9:.1f} GB")
    ref = RefLib()
    threads = os.cpu_count() or 1
    ref.set_threads(threads)
    sim = ref.sim(REF_CFG.format(nx=n, ny=n, nz=n, tau=tau))
    try:
        sim.shear_wave()
        for _ in range(max(1, warmup)):
            sim.run(1)
        t0 = time.perf_counter()
        sim.run(steps)
        dt = time.perf_counter() - t0
    finally:
        sim.close()
    cells = n ** 3
    return (cells * steps / dt / 1e6,
            f"reference Simulation::step (fluid, coupling off) on the full {n}x{n}x{n} periodic block, "
            f"{steps} timed steps after {max(1, warmup)} warm-up, shear-wave init, OpenMP, "
            f"{cpu_model()}", threads, dt / steps)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" x{os.cpu_count()}"
    except OSError:
        pass
    return f"{os.cpu_count()} host CPUs"


def arm_config(n, N, tau, halo):
    """The `config` object both arms print (the reference arm times the same workload)."""
    cells = n ** 3
    return {"workload": (f"config 2: pure-fluid D3Q19 SRT {n}^3 periodic, 1 GPU" if N == 1 else
                         f"config 4: pure-fluid D3Q19 SRT weak scaling {n}^3 per GPU, "
                         f"{n}x{n}x{n * N} periodic z-slabs"),
            "tau": tau, "cells_per_gpu": cells, "parallelism": f"z-slab x{N}",
            "l2": f"inputs larger than L2 ({2 * 19 * 8 * cells / 1e9:.1f} GB PDF working set)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    try:
        from oracle.pyoracle import REF_SO
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        mlups, sample, threads, per_step = reference_sample(args.n, args.tau, args.steps, args.warmup)
    except FileNotFoundError as e:
        print(json.dumps({"impl": "reference", "unavailable": f"reference build missing: {e}"}))
        return 0
    except MemoryError as e:  # the host cannot hold the full block: said so, never a smaller domain
        print(json.dumps({"impl": "reference", "unavailable": str(e)}))
        return 0
    line = {"metric": METRIC, "value": round(mlups, 3), "unit": "MLUPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(per_step * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (shear-wave initial state, validation.cpp:46-63)", "impl": "reference",
            "config": arm_config(args.n, args.gpus, args.tau, None),
            "cpu_baseline": {"value": round(mlups, 3), "unit": "MLUPS", "cores": threads,
                             "kind": "reference", "sample": sample},
            "e2e": {"value": round(mlups, 3), "unit": "MLUPS", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# --------------------------------------------------------------------------- coupled step
CONFIG3 = ('{"scenario":"fluidized_bed_dense","domain":[256,256,256],"particles":{"count":10000},'
           '"physical":{"diameter_cells":10},"fluid":{"bc":{"xm":"no_slip","xp":"no_slip",'
           '"ym":"no_slip","yp":"no_slip","zm":"velocity","zp":"pressure"}},'
           '"dem":{"k_n":230,"d_n":520,"k_t":65,"d_t":260,"subcycles":10}}')
CATS = ("PSM", "PSM-comm", "mapping", "setU", "redF", "PD", "PD-comm", "other")


def config3(blocks=(1, 1, 1), workers=1):
    c = json.loads(CONFIG3)
    c["blocks"], c["workers"] = list(blocks), workers
    return json.dumps(c)


REPS = 3  # best of >= 3 repetitions, the reference's own perf protocol (perf.cpp:104)


def _best_of(sim, steps, reps=REPS):
    """Run `reps` repetitions of `steps` coupled steps; (seconds, categories) of the fastest
    and the median wall time. Host-side phases (the reference's DEM and messaging on 8
    worker threads with nested OpenMP teams) see transient scheduling noise of up to +40 %
    on a shared host; the best repetition is the reference's reporting rule."""
    runs = []
    for _ in range(reps):
        sim.reset_timers()
        t0 = time.perf_counter()
        sim.run(steps)
        runs.append((time.perf_counter() - t0, sim.timings()))
    runs.sort(key=lambda r: r[0])
    return runs[0][0], runs[0][1], runs[len(runs) // 2][0]


def coupled_step(steps, with_reference, ref_steps=1, blocks=(1, 1, 1), workers=1):
    """Config 3: ~10^4 spheres d = 10 in 256^3, bed BCs, four-way coupled
    with the reference's host DEM. GPU side through the drop-in build (the reference
    Simulation with its fluid/coupling operators on liblbg); the same config on the
    unmodified reference (oracle/_ref, OpenMP on all host cores) for comparison. Times are
    the reference's own per-category wall-clock TimingReport (perf.hpp:17-51), best of
    REPS repetitions for both (perf.cpp:104)."""
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import dropin
    cfg = config3(blocks, workers)
    out = {"workload": "config 3: 10^4 spheres (d = 10) in 256^3, no-slip walls, velocity inflow, "
                       "pressure outflow, 10 DEM sub-cycles per fluid step (host DEM = reference code)",
           "blocks": list(blocks), "workers": workers, "repetitions": REPS}
    for mode in ("scratch", "fused"):
        # scratch: reference semantics, partials bitwise (PARITY reduction);
        # fused: force/torque summed inside the PSM kernel (FAST, tolerance-level partials)
        os.environ["LBDEM_GPU_FORCE"] = mode
        sim = dropin.DropinSim(cfg, (256, 256, 256))
        sim.run(1)  # warm-up (allocations, first mapping)
        dt, cat, med = _best_of(sim, steps)
        rec = {"ms_per_step": round(dt * 1e3 / steps, 2), "median_ms_per_step": round(med * 1e3 / steps, 2),
               "steps": steps,
               "categories_ms_per_step": {c: round(v * 1e3 / steps, 3) for c, v in zip(CATS, cat)},
               "gpu_side_ms_per_step": round(sum(cat[i] for i in (0, 1, 2, 3, 4)) * 1e3 / steps, 3),
               "particles": len(sim.particles()),
               "mlups": round(256 ** 3 * steps / dt / 1e6, 1)}
        sim.close()
        if mode == "scratch":
            out.update(rec)
        else:
            out["fused_force_mode"] = rec
    os.environ.pop("LBDEM_GPU_FORCE", None)
    if with_reference:
        from oracle.pyoracle import RefLib
        ref = RefLib()
        # all host cores: OpenMP teams inside each block worker share them
        threads = max(1, (os.cpu_count() or 1) // max(1, workers))
        ref.set_threads(threads)
        rs = ref.sim(cfg)
        rdt, rc, rmed = _best_of(rs, ref_steps)
        out["reference"] = {"ms_per_step": round(rdt * 1e3 / ref_steps, 1),
                            "median_ms_per_step": round(rmed * 1e3 / ref_steps, 1), "steps": ref_steps,
                            "repetitions": REPS, "threads": threads * max(1, workers), "workers": workers,
                            "omp_threads_per_worker": threads, "kind": "reference",
                            "categories_ms_per_step": {c: round(v * 1e3 / ref_steps, 2) for c, v in zip(CATS, rc)}}
        out["speedup_vs_reference"] = round(out["reference"]["ms_per_step"] / out["ms_per_step"], 2)
    return out


CONFIG5_1GPU = ('{"scenario":"fluidized_bed_dense","domain":[512,512,512],"blocks":[1,1,1],"workers":1,'
                '"particles":{"count":12500},"physical":{"diameter_cells":10},'
                '"fluid":{"bc":{"xm":"no_slip","xp":"no_slip","ym":"no_slip","yp":"no_slip",'
                '"zm":"velocity","zp":"pressure"}},'
                '"dem":{"k_n":230,"d_n":520,"k_t":65,"d_t":260,"subcycles":10,"settle_subcycles":100}}')


def coupled_sweep_roofline(steps=10, warmup=3, cfg=None, n=256, label="config 3 bed (reference scenario "
                           "particles), one 256^3 block, tau 0.567416"):
    """Device-side roofline of the coupled fluid step on config 3's bed (one 256^3 block):
    the particle list is the reference scenario's own (drop-in construction, 10^4 spheres
    d = 10 after settling), mapped once (K3); each step is the bed BCs (K5) followed by the
    coupled sweep of the whole block — K1 over the fluid segments || K2 over the covered
    segments — and a swap. With one block and no halo, BCs-then-sweep equals the reference's
    inner / BC / outer order (the BCs read and write only src; the sweep writes only dst).
    Algorithmic bytes per step: 305 B per cell + 44 B per one-entry cell + 80 B per two-entry
    cell (btot 8; per entry b 8 + id 4 read, m 24 written; v evaluated from the snapshots),
    SURVEY §8(d). CUDA events on the block's stream; inputs (5.4 GB) exceed L2."""
    import numpy as np
    import torch

    from paper_2303_11811_b200 import lbdem
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import dropin
    sim = dropin.DropinSim(cfg or config3(), (n, n, n))
    rows = sim.particles()
    sim.close()
    r = 5.0  # physical.diameter_cells / 2
    snaps = {"id": rows[:, 0].astype(np.int32), "x": rows[:, 1:4].copy(), "r": np.full(len(rows), r),
             "f_r": np.full(len(rows), lbdem.f_of_r(r)), "u": rows[:, 4:7].copy(), "w": rows[:, 7:10].copy()}
    tau, u_in = 0.567416, 2.2472e-3
    blk = lbdem.Block((n, n, n), coupling=True)
    try:
        blk.fill_equilibrium(1.0, (0.0, 0.0, u_in))
        blk.map(snaps)
        blk.sync()
        cnt = blk.download_fraction()["count"]
        n1, n2 = int((cnt == 1).sum()), int((cnt == 2).sum())
        # the sweep's per-block kernel choice (lbg_sweep.cu, LBG_K12=1): the covered fraction of
        # the aligned 32-cell row segments against LBG_K12_SPLIT_BELOW (0.35)
        segs = cnt.reshape(n, n, -1, 32).max(axis=3) if n % 32 == 0 else None
        cov_frac = float((segs > 0).mean()) if segs is not None else None
        del cnt, segs
        F = lbdem.FaceBc
        spec = lbdem.BcSpec([F(lbdem.BcKind.no_slip)] * 4 +
                            [F(lbdem.BcKind.velocity, (0.0, 0.0, u_in)), F(lbdem.BcKind.pressure, rho=1.0)])
        p = lbdem.FluidParams(tau)
        box = lbdem.CellBox((0, 0, 0), (n, n, n))
        stream = torch.cuda.ExternalStream(blk.stream)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        bc_ms = sweep_ms = 0.0
        for it in range(warmup + steps):
            ev[0].record(stream)
            blk.apply_boundaries(spec, [1] * 6)
            ev[1].record(stream)
            blk.sweep(p, box)
            ev[2].record(stream)
            blk.swap()
            if it >= warmup:
                ev[2].synchronize()
                bc_ms += ev[0].elapsed_time(ev[1])
                sweep_ms += ev[1].elapsed_time(ev[2])
        blk.sync()
        # K3 mapping (lbg_map: snapshot H2D + binning + map_col_kernel + segment lists) and K4
        # PARITY reduction (lbg_reduce_hydro: walk kernel + partials D2H + unpacking), each
        # timed on its own after the sweeps: CUDA events on the block stream for the mapping,
        # host wall clock for the reduction call (it returns the partials to the host)
        import ctypes as C
        from paper_2303_11811_b200 import lbg as abi
        lib = abi.load()
        map_ms, red_ms = [], []
        arr, nsn = lbdem.snapshot_array(snaps)  # the C-ABI snapshot list, built once
        for _ in range(5):
            ev[0].record(stream)
            lbdem.check(lib.lbg_map(blk.h, arr, nsn, 8))
            ev[1].record(stream)
            ev[1].synchronize()
            map_ms.append(ev[0].elapsed_time(ev[1]))
        blk.sync()
        cap = len(rows) + 16
        hp_out = (abi.HydroPartial * cap)()
        nout = C.c_int()
        for _ in range(5):
            blk.sweep(p, box)  # refills the scratch the reduction consumes (and clears)
            blk.sync()
            t0 = time.perf_counter()
            lbdem.check(lib.lbg_reduce_hydro(blk.h, abi.REDUCE_PARITY, hp_out, cap, C.byref(nout)))
            red_ms.append((time.perf_counter() - t0) * 1e3)
        map_ms.sort()
        red_ms.sort()
        # lbg_map call on the block stream (its host-side staging — snapshot copy into pinned
        # memory, registration bound — included: the stream idles meanwhile); kernel-only times
        # are in the ncu launch lists (profiles/)
        aux = {"mapping_ms": round(map_ms[len(map_ms) // 2], 4), "reduce_hydro_wall_ms": round(red_ms[len(red_ms) // 2], 4),
               "partials": nout.value}
        if os.environ.get("AB_REDUCE"):
            # wall time of lbg_reduce_hydro (PARITY) after a sweep refilled the scratch:
            # kernels + D2H + host unpacking of the partials, through the raw C-ABI call
            import ctypes as C
            from paper_2303_11811_b200 import lbg as abi
            lib = abi.load()
            cap = len(rows) + 16
            out = (abi.HydroPartial * cap)()
            nout = C.c_int()
            red = []
            for _ in range(5):
                blk.sweep(p, box)
                blk.sync()
                t0 = time.perf_counter()
                lbdem.check(lib.lbg_reduce_hydro(blk.h, abi.REDUCE_PARITY, out, cap, C.byref(nout)))
                red.append((time.perf_counter() - t0) * 1e3)
            os.environ["AB_REDUCE_MS"] = ",".join(f"{v:.3f}" for v in red)
    finally:
        blk.close()
    cells = n ** 3
    algo = 305 * cells + 44 * n1 + 80 * n2
    sweep_ms /= steps
    pk = peaks()
    peak = pk["hbm_gbs"] if pk and pk.get("hbm_gbs") else 6650.0
    achieved = algo / (sweep_ms / 1e3) / 1e9
    split = cov_frac is not None and cov_frac < float(os.environ.get("LBG_K12_SPLIT_BELOW", "0.35"))
    kernels = ("K1 sweep_box_kernel over the fluid segments + K12 coupled_unified_pipe_kernel over the "
               "covered-segment list" if split else
               "K12 coupled_unified_pipe_kernel (fluid, one-entry and two-entry segments in one kernel)")
    # K3 mapping against HBM: 9 B per cell (count + btot, written for every cell) + 12 B per entry
    # (id 4, b 8; + the 4-byte entry-0 snapshot index) — an issue-bound kernel, so the fraction
    # says how far it is from streaming, not what bounds it
    map_bytes = 9 * cells + 12 * (n1 + 2 * n2) + 4 * (n1 + n2)
    aux["mapping_algorithmic_bytes"] = map_bytes
    aux["mapping_frac_of_hbm"] = round(map_bytes / (aux["mapping_ms"] / 1e3) / 1e9 / peak, 4)
    return {"workload": label,
            "kernels": kernels, "covered_segment_fraction": None if cov_frac is None else round(cov_frac, 4),
            **aux,
            "cells": cells, "one_entry_cells": n1, "two_entry_cells": n2,
            "algorithmic_bytes_per_step": algo, "sweep_ms": round(sweep_ms, 4), "bc_ms": round(bc_ms / steps, 4),
            "mlups": round(cells / (sweep_ms / 1e3) / 1e6, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4)}}


def coupled_b0_roofline(n=512, tau=0.8, steps=10, warmup=3):
    """Config 2's second case: the same 512^3 periodic shear wave through the
    COUPLED sweep with no particles (coupling:true, P = 0) — psm_collide_stream's count == 0
    branch for every cell (psm.cpp:218-262). The mapping of an empty list zero-fills count and
    btot; the sweep is then K1 reading each cell's count (305 B per cell: 304 + 1 B count).
    CUDA events on the block's stream; inputs (43 GB) exceed L2."""
    import torch

    from paper_2303_11811_b200 import lbdem
    blk = lbdem.Block((n, n, n), coupling=True)
    try:
        blk.init_shear_wave((n, n, n))
        blk.set_periodic_wrap((1, 1, 1))
        blk.map([])
        p = lbdem.FluidParams(tau)
        box = lbdem.CellBox((0, 0, 0), (n, n, n))
        stream = torch.cuda.ExternalStream(blk.stream)
        for _ in range(warmup):
            blk.sweep(p, box)
            blk.swap()
        blk.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            blk.sweep(p, box)
            blk.swap()
        e1.record(stream)
        e1.synchronize()
        blk.sync()
        ms = e0.elapsed_time(e1) / steps
    finally:
        blk.close()
    cells = n ** 3
    algo = 305 * cells
    pk = peaks()
    peak = pk["hbm_gbs"] if pk and pk.get("hbm_gbs") else 6650.0
    achieved = algo / (ms / 1e3) / 1e9
    return {"workload": f"config 2, coupling:true with P = 0: {n}^3 periodic shear wave, tau {tau}",
            "cells": cells, "algorithmic_bytes_per_step": algo, "sweep_ms": round(ms, 4),
            "mlups": round(cells / (ms / 1e3) / 1e6, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4)}}


def aa_roofline(n=512, tau=0.8, steps=10, warmup=4):
    """Config 2 with the AA-pattern in-place streaming (lbg_set_streaming(LBG_STREAM_AA)): the
    same 512^3 periodic shear wave and 304 B per LUP in ONE PDF buffer (the second is released:
    half the HBM). Even step counts (both AA phases per pair of steps); CUDA events on the
    block's stream."""
    import ctypes as C

    import torch

    from paper_2303_11811_b200 import lbdem
    from paper_2303_11811_b200 import lbg as abi
    blk = lbdem.Block((n, n, n))
    try:
        mem = C.c_longlong()
        abi.load().lbg_block_info(blk.h, None, None, None, C.byref(mem))
        mem_ab = mem.value
        blk.init_shear_wave((n, n, n))
        blk.set_periodic_wrap((1, 1, 1))
        blk.set_streaming(abi.STREAM_AA)
        abi.load().lbg_block_info(blk.h, None, None, None, C.byref(mem))
        p = lbdem.FluidParams(tau)
        box = lbdem.CellBox((0, 0, 0), (n, n, n))
        stream = torch.cuda.ExternalStream(blk.stream)
        for _ in range(warmup):
            blk.sweep(p, box)
            blk.swap()
        blk.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            blk.sweep(p, box)
            blk.swap()
        e1.record(stream)
        e1.synchronize()
        blk.sync()
        ms = e0.elapsed_time(e1) / steps
    finally:
        blk.close()
    cells = n ** 3
    pk = peaks()
    peak = pk["hbm_gbs"] if pk and pk.get("hbm_gbs") else 6650.0
    achieved = BYTES_PER_LUP * cells / (ms / 1e3) / 1e9
    return {"workload": f"config 2 with AA in-place streaming: {n}^3 periodic shear wave, tau {tau}",
            "device_bytes": mem.value, "device_bytes_double_buffer": mem_ab,
            "sweep_ms": round(ms, 4), "mlups": round(cells / (ms / 1e3) / 1e6, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4)}}


def pcie_rates(host, device, nbytes=2 << 30):
    """PCIe copy rates (GB/s) on `nbytes` of the pinned host buffer `host` (numpy, float64):
    H2D alone, D2H alone, and both directions at once (separate streams) — the floor the
    streamed job's e2e is measured against."""
    import torch
    flat = host.reshape(-1)
    cnt = min(nbytes // 8, flat.size // 2)
    hb = torch.from_numpy(flat[: 2 * cnt])
    d1 = torch.empty(cnt, dtype=torch.float64, device=f"cuda:{device}")
    d2 = torch.empty(cnt, dtype=torch.float64, device=f"cuda:{device}")
    s1, s2 = torch.cuda.Stream(device), torch.cuda.Stream(device)
    keep = hb[cnt:].clone()  # the D2H legs overwrite the buffer's second half: restore it

    def timed(fn):
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize(device)
        return time.perf_counter() - t0

    d1.copy_(hb[:cnt], non_blocking=True)  # warm
    h2d = timed(lambda: d1.copy_(hb[:cnt], non_blocking=True))
    d2h = timed(lambda: hb[cnt:].copy_(d2, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(hb[:cnt], non_blocking=True)
        with torch.cuda.stream(s2):
            hb[cnt:].copy_(d2, non_blocking=True)
    bt = timed(both)
    hb[cnt:].copy_(keep)
    gb = cnt * 8 / 1e9
    return {"h2d_gbs": round(gb / h2d, 1), "d2h_gbs": round(gb / d2h, 1), "both_gbs_each": round(gb / bt, 1),
            "sample_gb": round(gb, 2)}


def e2e_record(args, n, pdf_bytes, e2e_mlups, loop_mlups, job_mlups, finite, numa_cpus, pcie=None, job_s=None):
    """The e2e object: with one GPU the streamed job (lbg_run_host; its H2D carries the 19 x nz
    interior z-planes incl. their x/y ghost rows, its D2H the same planes plus the 48-byte error
    counters), the unpipelined job beside it; with N > 1 the unpipelined job per rank."""
    unpiped = {"value": round(e2e_mlups, 1),
               "h2d_bytes_per_step": round(pdf_bytes / args.steps),
               "d2h_bytes_per_step": round(pdf_bytes / args.steps) + 24,
               "how": (f"job of {args.steps} steps through the C-ABI with host buffers: lbg_upload_src "
                       "from pinned host memory (reference layout), per step sweep [+ halo] + swap + "
                       "lbg_sync (error-counter D2H, NumericError check), lbg_download_src; wall clock, "
                       "max over ranks"),
               "steady_state_loop_mlups": round(loop_mlups, 1)}
    common = {"result_finite": finite, "host_buffer_numa_cpus": len(numa_cpus) if numa_cpus else None}
    if job_mlups is None:
        return {"value": unpiped["value"], "unit": "MLUPS", "h2d_bytes_per_step": unpiped["h2d_bytes_per_step"],
                "d2h_bytes_per_step": unpiped["d2h_bytes_per_step"], "how": unpiped["how"],
                "steady_state_loop_mlups": unpiped["steady_state_loop_mlups"], **common}
    moved = 8 * 19 * n * (n + 2) * (n + 2)
    return {"value": round(job_mlups, 1), "unit": "MLUPS",
            "h2d_bytes_per_step": round(moved / args.steps),
            "d2h_bytes_per_step": round((moved + 48) / args.steps),
            "how": (f"job of {args.steps} steps through the C-ABI with host buffers: lbg_run_host on the "
                    "pinned host PdfField (reference layout) — H2D of the state, the K fused sweeps and "
                    "D2H of the final state pipelined over 16-plane z-slabs on separate streams (both PCIe "
                    "directions at once; with N GPUs one NCCL seam exchange per step), then the accumulated "
                    "NumericError check (error-counter D2H); wall clock, max over ranks; interior result "
                    "bitwise that of the unpipelined job (tests/test_gpu_job.py, test_gpu_multi.py)"),
            "unpipelined": unpiped,
            # the PCIe floor: H2D and D2H of the field overlap, so the job cannot beat the
            # field's bytes at the both-directions rate (per rank)
            "pcie": (None if pcie is None or job_s is None else
                     {**pcie, "job_gbs_each": round(moved / job_s / 1e9, 1),
                      "frac_of_both": round(moved / job_s / 1e9 / pcie["both_gbs_each"], 3)}),
            **common}


def host_mem_available():
    """MemAvailable of this host in bytes (None if unknown)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def gpu_local_cpus(device):
    """Host CPUs NVML reports closest to CUDA device `device` (its NUMA node), matched by PCI
    bus id; None if unknown. The e2e job pins its host PdfField from a thread bound to them,
    so the pages and the DMA stay on the GPU's socket."""
    try:
        import pynvml
        import torch
        pr = torch.cuda.get_device_properties(device)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        words = ((os.cpu_count() or 64) + 63) // 64
        mask = pynvml.nvmlDeviceGetCpuAffinity(h, words)
        cpus = {64 * w + b for w, m in enumerate(mask) for b in range(64) if (m >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:  # noqa: BLE001 — no NVML / no PCI info: leave the affinity alone
        return None


SPEC_HBM_GBS = 8000.0  # B200 HBM3e datasheet figure (report against it too)
NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (B200_PROFILING.md)


def halo_record(halo, n, ms_step, tm, steps):
    """PDF halo per GPU and step: 5 inbound q per face cell, from each of the
    two slab neighbours, 8 B each — and the NVLink fraction it needs. With the NCCL halo the
    comm-stream time (pack, ncclSend/Recv, unpack; CUDA events) is measured and overlapped
    with the inner sweep; with P2P the stores are issued by the outer sweep kernel itself, so
    the transfer has no separate phase."""
    nbytes = 2 * 5 * n * n * 8
    rec = {"mode": halo, "bytes_per_gpu_per_step": nbytes,
           "nvlink_gbs_needed_at_step_rate": round(nbytes / (ms_step / 1e3) / 1e9, 2),
           "frac_of_nvlink_needed": round(nbytes / (ms_step / 1e3) / 1e9 / NVLINK_GBS, 5)}
    comm = tm.get("PSM-comm")
    if comm and comm[1]:
        ms = comm[0] / steps
        rec["comm_stream_ms_per_step"] = round(ms, 4)
        rec["achieved_gbs_during_comm"] = round(nbytes / (ms / 1e3) / 1e9, 1)
        rec["frac_of_nvlink_during_comm"] = round(nbytes / (ms / 1e3) / 1e9 / NVLINK_GBS, 4)
    return rec


# --------------------------------------------------------------------------- GPU path
def run_lbg(args):
    import torch
    import torch.distributed as dist

    from paper_2303_11811_b200 import lbdem

    rank, world, local = dist_env()
    N = world
    share = os.environ.get("LBG_BENCH_SHARE_GPUS") == "1"
    if share:
        # functional check of an N-rank ring on fewer GPUs (ranks share devices, so the
        # plumbing runs on gloo — NCCL refuses two ranks per GPU — and the timings are not
        # per-GPU numbers)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2303_11811_b200.driver import FluidStepper, SlabDecomposition
    n = args.n
    dims = (n, n, n)
    domain = (n, n, n * N)
    p = lbdem.FluidParams(args.tau)
    dec = SlabDecomposition(domain, N, axis=2, periodic=(1, 1, 1))
    uid = [lbdem.comm_unique_id() if (rank == 0 and N > 1) else None]
    if N > 1:
        dist.broadcast_object_list(uid, src=0)

    def allgather(b: bytes):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    # x, y (and z on one GPU) are periodic and spanned by the block: wrapped in-kernel;
    # z between GPUs: NCCL halo behind the inner sweep, or the outer sweep's P2P stores
    halo = args.halo
    st = None
    if N > 1 and halo == "p2p":
        # the P2P mapping is opened per rank after the handle exchange; if any rank cannot
        # map its neighbours, every rank falls back to the NCCL halo (decided collectively)
        err = None
        try:
            st = FluidStepper(dec, rank, p, device=local, uid=uid[0], halo="p2p", allgather=allgather)
        except Exception as e:  # noqa: BLE001 — reported, then the NCCL path is used
            err = f"{type(e).__name__}: {e}"
        errs = [x for x in allgather(err) if x]
        if errs:
            if rank == 0:
                print(f"P2P halo unavailable ({errs[0]}); using the NCCL halo", file=sys.stderr)
            if st is not None:
                st.block.close()
                st = None
            halo = "nccl"
    if st is None:
        st = FluidStepper(dec, rank, p, device=local, uid=uid[0], halo=halo, allgather=allgather)
    blk = st.block
    blk.init_shear_wave(domain)
    if N > 1:
        torch.cuda.synchronize()
        dist.barrier()
        st.prime()
        dist.barrier()
    step = st.step

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if share else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    blk.sync()
    stream = torch.cuda.ExternalStream(blk.stream, device=torch.device("cuda", local))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    # ---- device-timed region
    barrier()
    blk.set_timing(True)
    blk.timings()  # clear
    l0 = lbdem.launch_count()
    with ClockSampler(local) as clk:
        barrier()  # all ranks' samplers are running
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        e1.synchronize()
    launches = lbdem.launch_count() - l0
    tm = blk.timings()
    blk.set_timing(False)
    blk.sync()  # stability check (NumericError would raise here)
    barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms_total / args.steps
    cells = n * n * n
    mlups = cells * N * args.steps / (ms_total / 1e3) / 1e6

    sweep_ms, sweep_n = tm["PSM"]
    sweep_ms_per_step = sweep_ms / args.steps
    achieved = BYTES_PER_LUP * cells / (sweep_ms_per_step / 1e3) / 1e9  # GB/s
    pk = peaks()
    peak, peak_src = (pk["hbm_gbs"], "measured") if pk and pk.get("hbm_gbs") else (6650.0, "fallback")
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            if tj.get("n") == n:
                traffic = tj.get("bytes_per_launch")
        except Exception:
            traffic = None

    # ---- end to end through the C-ABI with host buffers: the job a caller with a host
    # PdfField runs — upload the state from pinned host memory (reference idx() layout),
    # K steps each closed by the reference's end-of-operator check (lbg_sync: D2H of the
    # error counters, raises NumericError), download the final state to the host buffer.
    import ctypes as C
    import numpy as np
    from paper_2303_11811_b200 import lbg as abi
    pdf_bytes = 8 * 19 * (n + 2) ** 3
    # every rank of this host pins its own full host PdfField: run the job only if they all fit
    # comfortably in the host's available memory (an 8-GPU box must not be driven out of RAM)
    local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    avail = host_mem_available()
    fits = avail is None or local_ranks * pdf_bytes <= 0.6 * avail
    fits = all(allgather(fits)) if N > 1 else fits
    e2e_mlups = loop_mlups = job_mlups = job_s = pcie = None
    finite = None
    numa_cpus = None
    saved_affinity = os.sched_getaffinity(0)
    if fits and os.environ.get("LBG_BENCH_NUMA", "1") != "0":
        numa_cpus = gpu_local_cpus(local)
        if numa_cpus:
            os.sched_setaffinity(0, numa_cpus)
    if fits:
        hp = C.c_void_p()
        lbdem.check(abi.load().lbg_host_alloc(pdf_bytes, C.byref(hp)))
        host = np.ctypeslib.as_array(C.cast(hp, C.POINTER(C.c_double)), shape=(19, n + 2, n + 2, n + 2))
        lbdem.check(abi.load().lbg_download_src(blk.h, hp))  # the current state as the job's input
        if dec.axis == 2:
            # the streamed job (lbg_run_host): the same upload, K steps and download, pipelined
            # over z-slabs so both PCIe directions and the sweeps overlap (one GPU: z wrapped
            # in-kernel; N GPUs: z-slabs, whose seam planes take one NCCL halo exchange per
            # step — a P2P-mode block gets an NCCL comm for it); the unpipelined job below
            # runs afterwards for comparison, continuing from its result (same work)
            if N > 1 and st.p2p:
                blk.comm_init(N, rank, uid[0], axis=2, periodic=(1, 1, 1))
            # its slab staging (6 x 0.64 GB) is allocated, and with N GPUs the NCCL seam
            # connections are set up, by one untimed 1-step job, as the unpipelined job's
            # staging is by the untimed download above
            blk.run_host(p, host, 1)
            barrier()
            t0 = time.perf_counter()
            blk.run_host(p, host, args.steps)
            t1 = time.perf_counter()
            barrier()
            job_s = max_over_ranks(t1 - t0)
            job_mlups = cells * N * args.steps / job_s / 1e6
            try:
                pcie = pcie_rates(host, local)
            except Exception:  # noqa: BLE001 — a report, not the measurement
                pcie = None
        barrier()
        t0 = time.perf_counter()
        lbdem.check(abi.load().lbg_upload_src(blk.h, hp))
        tl0 = time.perf_counter()
        for _ in range(args.steps):
            step()
            blk.sync()  # lbg_sync: D2H of the 3 error counters, raises NumericError/SyncError
        tl1 = time.perf_counter()
        lbdem.check(abi.load().lbg_download_src(blk.h, hp))
        t1 = time.perf_counter()
        barrier()
        e2e_s = max_over_ranks(t1 - t0)
        loop_s = max_over_ranks(tl1 - tl0)
        e2e_mlups = cells * N * args.steps / e2e_s / 1e6
        loop_mlups = cells * N * args.steps / loop_s / 1e6
        finite = bool(np.isfinite(host[:, n // 2, n // 2, 1:5]).all())
        del host
        abi.load().lbg_host_free(hp)
    os.sched_setaffinity(0, saved_affinity)  # the CPU baseline below uses every host core

    out = None
    if rank == 0:
        cpu = None
        if N == 1 and not args.no_cpu_baseline:
            try:
                c_mlups, sample, threads, _ = reference_sample(n, args.tau, args.cpu_steps)
                cpu = {"value": round(c_mlups, 3), "unit": "MLUPS", "cores": threads,
                       "kind": "reference", "sample": sample}
            except Exception as e:  # noqa: BLE001
                cpu = {"value": None, "unit": "MLUPS", "cores": 0, "kind": "reference",
                       "sample": f"unavailable: {e}"}
        out = {
            "metric": METRIC, "value": round(mlups, 1), "unit": "MLUPS", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (shear-wave initial state, validation.cpp:46-63, device-initialised)",
            "config": arm_config(n, N, args.tau, halo),
            "mlups_per_gpu": round(mlups / N, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "sweep_box_kernel<false,false> (K1 fused pull stream-collide)",
                         "bytes_per_lup": BYTES_PER_LUP, "peak_source": peak_src,
                         "frac_of_spec_8000": round(achieved / SPEC_HBM_GBS, 4),
                         "sweep_ms_per_step": round(sweep_ms_per_step, 4),
                         "sweep_launches": sweep_n},
            "hbm_roofline_frac_of_step": round(BYTES_PER_LUP * cells / (ms_step / 1e3) / 1e9 / peak, 4),
            "timings_ms_per_step": {k: round(v[0] / args.steps, 4) for k, v in tm.items() if v[1]},
            "halo": (None if N == 1 else halo_record(halo, n, ms_step, tm, args.steps)),
            "e2e": (e2e_record(args, n, pdf_bytes, e2e_mlups, loop_mlups, job_mlups, finite, numa_cpus, pcie, job_s)
                    if e2e_mlups is not None else
                    {"value": None, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                     "skipped": (f"{local_ranks} host PdfFields of {pdf_bytes / 1e9:.1f} GB exceed 60 % of the "
                                 f"host's available memory ({(avail or 0) / 1e9:.0f} GB)")}),
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
    blk.close()
    if rank == 0 and N == 1 and not args.no_coupled:
        try:
            out["coupled_b0"] = coupled_b0_roofline(n, args.tau)
        except Exception as e:  # noqa: BLE001
            out["coupled_b0"] = {"unavailable": f"{type(e).__name__}: {e}"}
        try:
            out["aa_streaming"] = aa_roofline(n, args.tau)
        except Exception as e:  # noqa: BLE001
            out["aa_streaming"] = {"unavailable": f"{type(e).__name__}: {e}"}
    if rank == 0:
        if N == 1 and not args.no_coupled:
            try:
                # the reference's own parallelism lever: blocks with one worker thread each (host
                # DEM per block in parallel) — 2x2x4 / 16 workers on a host with >= 16 CPUs (one
                # polling worker per CPU; 8.6-11 ms vs 11.6-11.7 for 2x2x2 / 8, profiles/
                # r02_c3blocks4.log), else 2x2x2; the same blocks/workers for the reference run
                cpus = os.cpu_count() or 8
                blocks, workers = ((2, 2, 4), 16) if cpus >= 16 else ((2, 2, 2), min(8, cpus))
                out["coupled_step"] = coupled_step(args.coupled_steps, not args.no_cpu_baseline, ref_steps=1,
                                                   blocks=blocks, workers=workers)
                single = coupled_step(args.coupled_steps, False)
                out["coupled_step"]["single_block"] = {k: single[k] for k in (
                    "ms_per_step", "categories_ms_per_step", "gpu_side_ms_per_step", "fused_force_mode")}
                out["coupled_step"]["psm_sweep"] = coupled_sweep_roofline()
                # config 5's dilute bed (12,500 spheres in 512^3, 4.9 % solid) as one block
                out["coupled_step"]["psm_sweep_config5"] = coupled_sweep_roofline(
                    cfg=CONFIG5_1GPU, n=512, label="config 5 bed (12,500 spheres d = 10 after 100 settling "
                    "sub-cycles), one 512^3 block, tau 0.567416")
            except Exception as e:  # noqa: BLE001
                out["coupled_step"] = {"unavailable": f"{type(e).__name__}: {e}"}
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_lbg(args)


if __name__ == "__main__":
    sys.exit(main())
