"""Parity at BASELINE.json's full sizes.

* config 3 — the 10^4-sphere bed in 256^3 (bench.py CONFIG3, one block): the drop-in (the
  reference Simulation with its fluid/coupling operators on liblbg) and the unmodified
  reference (oracle/_ref) from the same config, two coupled steps; every PDF and particle
  state bitwise equal. This runs the mapping (~7 M fraction entries), the PSM sweep with
  two-entry cells, the bed BCs and the PARITY force reduction at the benchmarked size.
* config 2 — the 512^3 periodic shear-wave block of bench.py: one step on the GPU, then the
  oracle (oracle/lbm_oracle.c, collide_stream) replays 16^3 windows — corners wrapping on all
  three axes, an x-wrap straddle and interior windows — from the GPU's own pre-step state;
  the GPU's post-step populations are bitwise the oracle's. Over ten steps the total mass
  (compensated device sum) is conserved to 1e-12 relative (test_lattice_lbm.cpp:303-322 at
  full size).
Host memory: the 512^3 check holds one 20.6 GB PDF field on the host at a time.
"""
import json
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, equal_bits

pytestmark = pytest.mark.gpu


def mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def test_config3_full_bed_two_steps_bitwise(ref):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import torch  # noqa: F401  (CUDA plumbing)
    import bench
    import dropin
    dropin.load()
    cfg = bench.config3()
    a = dropin.DropinSim(cfg, (256, 256, 256))
    b = ref.sim(cfg)
    try:
        pa0, pb0 = a.particles(), b.particles()
        assert len(pa0) == 10000 and equal_bits(pa0, pb0)
        a.run(2)
        b.run(2)
        assert equal_bits(a.particles(), b.particles())
        assert equal_bits(a.pdfs(), b.pdfs())
    finally:
        a.close()


WIN = 16


def _window(full, lo, n):
    """(19, w+2, w+2, w+2) block of a periodic n^3 field (reference layout, ghosts at 0 and
    n+1) around the interior window [lo, lo + WIN)^3, halo taken from the periodic image —
    what fill_periodic_ghosts (boundary.cpp:98-137) gives a block of that size."""
    idx = [np.arange(lo[d] - 1, lo[d] + WIN + 1) % n + 1 for d in range(3)]  # x, y, z
    return np.ascontiguousarray(full[np.ix_(np.arange(19), idx[2], idx[1], idx[0])])


def test_config2_512_windows_bitwise_and_mass(gpu, oracle):
    n = 512
    need = 8 * 19 * (n + 2) ** 3
    if mem_available() < 1.4 * need:
        pytest.skip(f"needs {1.4 * need / 1e9:.0f} GB of host memory for one {n}^3 PDF field")
    tau = 0.8
    blk = gpu.Block((n, n, n))
    try:
        blk.set_periodic_wrap((1, 1, 1))
        blk.init_shear_wave((n, n, n))
        p = gpu.FluidParams(tau)
        box = gpu.CellBox((0, 0, 0), (n, n, n))
        m0 = blk.observe()["mass"]
        blk.sweep(p, box)
        blk.swap()
        blk.sync()
        wins = [(0, 0, 0), (n - WIN, n - WIN, n - WIN), (n - WIN // 2, 100, 300), (250, n - 3, 7),
                (131, 257, 389)]
        old = blk.download_dst()  # the pre-step state (the swap made it dst)
        src_w = [_window(old, lo, n) for lo in wins]
        del old
        new = blk.download_src()
        got = [np.ascontiguousarray(_window(new, lo, n)[:, 1:-1, 1:-1, 1:-1]) for lo in wins]
        del new
        dims = (WIN, WIN, WIN)
        for lo, s, g in zip(wins, src_w, got):
            d = np.zeros_like(s)
            oracle.collide_stream(dims, s, d, tau, (0.0, 0.0, 0.0), (0, 0, 0), dims)
            assert equal_bits(g, d[:, 1:-1, 1:-1, 1:-1]), f"window at {lo}"
        for _ in range(9):
            blk.sweep(p, box)
            blk.swap()
        blk.sync()
        m1 = blk.observe()["mass"]
        assert abs(m1 - m0) <= 1e-12 * abs(m0), (m0, m1)
    finally:
        blk.close()


def test_config2_aa_streaming_full_size_bitwise(gpu):
    """The AA in-place layout at config 2's size: the 512^3 periodic shear wave stepped 4 times
    in one buffer and 4 times double-buffered from the same device-initialised state give
    bitwise equal per-cell moments (rho and the bare momentum, lbg_moments) over all 1.3e8
    cells — an even step count, so the AA buffer holds the double-buffer state S0 — and, after
    a fifth (odd) step, bitwise equal populations in sampled planes of the downloaded src."""
    from paper_2303_11811_b200 import lbg
    n = 512
    if mem_available() < 60e9:
        pytest.skip("needs ~60 GB of host memory for two moment arrays and one PDF field")
    p = gpu.FluidParams(0.8)
    box = gpu.CellBox((0, 0, 0), (n, n, n))
    out = {}
    for mode in ("ab", "aa"):
        blk = gpu.Block((n, n, n))
        try:
            blk.init_shear_wave((n, n, n))
            blk.set_periodic_wrap((1, 1, 1))
            if mode == "aa":
                blk.set_streaming(lbg.STREAM_AA)
            for _ in range(4):
                blk.sweep(p, box)
                blk.swap()
            assert blk.sync()["unstable"] == 0
            mom = blk.moments()
            out[mode] = np.ascontiguousarray(mom).view(np.uint64).copy()
            del mom
            blk.sweep(p, box)
            blk.swap()
            f = blk.download_src()
            out[mode + "_planes"] = np.ascontiguousarray(f[:, [1, 2, n // 2, n - 1, n], :, :]).copy()
            del f
        finally:
            blk.close()
    assert np.array_equal(out["ab"], out["aa"])
    assert np.array_equal(out["ab_planes"].view(np.uint64), out["aa_planes"].view(np.uint64))
