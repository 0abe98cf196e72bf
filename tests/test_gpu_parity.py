"""GPU parity: every liblbg operator against the CPU oracle on identical inputs.

The bar is bitwise equality (fp64, --fmad=false kernels vs the -ffp-contract=off reference
restatement) for PDFs, ghost fills, BC values, fraction fields, solid velocities, momentum
scratch and PARITY-mode force partials; FAST-mode partials use the L1-mass tolerance of
SURVEY.md §8(c): |dF| <= 1e-12 * sum |m|.
"""
import numpy as np
import pytest

from conftest import W, equal_bits, interior, n_bit_mismatch, random_pdf
from oracle.pyoracle import make_snapshots, new_fraction, new_scratch, new_svel

pytestmark = pytest.mark.gpu

ALL_P = (1, 1, 1)


def run_oracle_step(oracle, dims, src, tau, fext, periodic=ALL_P, box=None):
    src = src.copy()
    dst = np.zeros_like(src)
    oracle.fill_periodic(dims, src, periodic)
    lo, hi = box if box else ((0, 0, 0), dims)
    bad = oracle.collide_stream(dims, src, dst, tau, fext, lo, hi)
    return src, dst, bad


@pytest.mark.parametrize("dims,fext", [((8, 8, 8), (1e-5, 0.0, -2e-5)),
                                       ((13, 7, 5), (0.0, 0.0, 0.0)),
                                       ((40, 3, 9), (2e-6, 1e-6, 0.0))])
def test_fused_sweep_bitwise(gpu, oracle, dims, fext):
    src0 = random_pdf(dims, seed=29)
    tau = 0.8
    src_o, dst_o, bad = run_oracle_step(oracle, dims, src0, tau, fext)
    assert bad == 0
    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.fill_periodic(ALL_P, full=True)
    blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox((0, 0, 0), dims))
    blk.sync()
    assert equal_bits(blk.download_src(), src_o), "periodic ghost fill differs"
    got = blk.download_dst()
    assert n_bit_mismatch(interior(got), interior(dst_o)) == 0


def test_sweep_sub_boxes_and_shell(gpu, oracle):
    dims = (20, 11, 9)
    tau, fext = 0.73, (0.0, 3e-6, 0.0)
    src0 = random_pdf(dims, seed=3)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    inner = ((1, 1, 1), (dims[0] - 1, dims[1] - 1, dims[2] - 1))
    oracle.collide_stream(dims, src_o, dst_o, tau, fext, *inner)
    shell = gpu.boundary_shell(dims)
    for b in shell:
        oracle.collide_stream(dims, src_o, dst_o, tau, fext, b.lo, b.hi)

    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.fill_periodic(ALL_P, full=True)
    p = gpu.FluidParams(tau, fext)
    blk.sweep(p, gpu.CellBox(*inner))
    blk.sweep_boxes(p, shell)
    blk.sync()
    assert equal_bits(interior(blk.download_dst()), interior(dst_o))


def test_unfused_stream(gpu, oracle):
    dims = (6, 6, 6)
    src0 = random_pdf(dims, seed=17)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    oracle.stream(dims, src_o, dst_o, (0, 0, 0), dims)
    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.fill_periodic(ALL_P, full=True)
    blk.stream_only(gpu.CellBox((0, 0, 0), dims))
    assert equal_bits(interior(blk.download_dst()), interior(dst_o))


@pytest.mark.parametrize("periodic", [(1, 1, 1), (1, 0, 1), (0, 1, 0), (0, 0, 1)])
def test_periodic_fill_full_bitwise_and_pull_only_equivalent(gpu, oracle, periodic):
    dims = (9, 5, 7)
    src0 = random_pdf(dims, seed=5)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, periodic)
    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.fill_periodic(periodic, full=True)
    assert equal_bits(blk.download_src(), src_o)
    # pull-only fill feeds the sweep exactly the same values
    tau, fext = 0.9, (0.0, 0.0, 1e-6)
    dst_o = np.zeros_like(src_o)
    oracle.collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims)
    blk.upload_src(src0)
    blk.fill_periodic(periodic, full=False)
    blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox((0, 0, 0), dims))
    blk.sync()
    if all(periodic):
        assert equal_bits(interior(blk.download_dst()), interior(dst_o))


@pytest.mark.parametrize("wrap", [(1, 1, 1), (1, 0, 1), (0, 1, 0), (0, 0, 1)])
@pytest.mark.parametrize("coupled", [False, True])
def test_in_kernel_periodic_wrap_bitwise(gpu, oracle, wrap, coupled):
    """lbg_set_periodic_wrap: wrapped pulls == pulls from periodically filled ghosts."""
    dims = (13, 9, 7)
    src0 = random_pdf(dims, seed=21)
    tau, fext = 0.77, (1e-6, 0.0, -2e-6)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    blk = gpu.Block(dims, coupling=coupled)
    if coupled:
        frac, sv = random_fraction(dims, seed=4)
        scr = new_scratch(dims)
        oracle.psm_collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims, frac, sv, scr)
        blk.upload_fraction(frac)
        blk.upload_solid_velocity(sv["v0"], sv["v1"])
    else:
        oracle.collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims)
    blk.upload_src(src0)
    blk.set_periodic_wrap(wrap)  # before the fill: the pull-only fill honours the wrap
    blk.fill_periodic(tuple(1 - w for w in wrap), full=False)
    blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox((0, 0, 0), dims))
    blk.sync()
    assert n_bit_mismatch(interior(blk.download_dst()), interior(dst_o)) == 0
    if coupled:
        m0, _ = blk.download_scratch()
        c = frac["count"]
        assert equal_bits(m0[c > 0], scr["m0"][c > 0])


@pytest.mark.parametrize("dims", [(64, 4, 3), (66, 5, 3), (127, 3, 4), (130, 6, 3)])
@pytest.mark.parametrize("wrap", [(0, 0, 0), (1, 1, 1), (1, 0, 0), (0, 1, 1)])
def test_sweep_warp_edges_bitwise(gpu, oracle, dims, wrap):
    """K1 at row lengths that end mid-warp / mid-pair, odd box origins and x-wrap on even and
    odd nx (with LBG_SWEEP_PAIR=1 — test_pair_kernel_variant — the 128-bit pair kernel:
    two cells per lane, x-neighbours by shuffle)."""
    src0 = random_pdf(dims, seed=dims[0])
    tau, fext = 0.81, (2e-6, -1e-6, 0.0)
    boxes = [((0, 0, 0), dims), ((1, 1, 1), tuple(d - 1 for d in dims)),
             ((3, 0, 1), (min(dims[0], 61), dims[1], dims[2]))]
    for lo, hi in boxes:
        src_o = src0.copy()
        oracle.fill_periodic(dims, src_o, ALL_P)
        dst_o = np.zeros_like(src_o)
        oracle.collide_stream(dims, src_o, dst_o, tau, fext, lo, hi)
        blk = gpu.Block(dims)
        blk.upload_src(src0)
        blk.set_periodic_wrap(wrap)
        blk.fill_periodic(tuple(1 - w for w in wrap), full=False)
        blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox(lo, hi))
        blk.sync()
        got = blk.download_dst()
        assert n_bit_mismatch(interior(got), interior(dst_o)) == 0, (lo, hi)


def test_pair_kernel_variant():
    """The same edge cases through the 128-bit pair kernel (selected per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, LBG_SWEEP_PAIR="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "test_gpu_parity.py::test_sweep_warp_edges_bitwise",
                        "test_gpu_parity.py::test_fused_sweep_bitwise",
                        "test_gpu_parity.py::test_unstable_cell_count_matches_reference"], env=env,
                       cwd=os.path.dirname(os.path.abspath(__file__)), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def bed_spec(gpu, zm_vel=(0.0, 0.0, 2.2472e-3), rho_out=1.0):
    spec = gpu.BcSpec()
    for f in range(4):
        spec.faces[f] = gpu.FaceBc(gpu.BcKind.no_slip)
    spec.faces[4] = gpu.FaceBc(gpu.BcKind.velocity, zm_vel)
    spec.faces[5] = gpu.FaceBc(gpu.BcKind.pressure, (0.0, 0.0, 0.0), rho_out)
    return spec


def spec_arrays(spec):
    kinds = [int(f.kind) for f in spec.faces]
    uw = np.array([f.u_wall for f in spec.faces], dtype=np.float64).ravel()
    rho = [f.rho for f in spec.faces]
    return kinds, uw, rho


@pytest.mark.parametrize("case", ["bed", "channel_y", "mixed_touch"])
def test_apply_boundaries_bitwise(gpu, oracle, case):
    dims = (7, 6, 8)
    src0 = random_pdf(dims, seed=41)
    if case == "bed":
        spec, touches, periodic = bed_spec(gpu), (1, 1, 1, 1, 1, 1), (0, 0, 0)
    elif case == "channel_y":
        spec = gpu.BcSpec()
        spec.faces[2] = gpu.FaceBc(gpu.BcKind.no_slip)
        spec.faces[3] = gpu.FaceBc(gpu.BcKind.velocity, (0.01, 0.0, 0.002))
        touches, periodic = (1, 1, 1, 1, 1, 1), (1, 0, 1)
    else:  # a block touching only some domain faces
        spec, touches, periodic = bed_spec(gpu, rho_out=1.01), (1, 0, 0, 1, 1, 0), (0, 0, 0)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, periodic)
    oracle.apply_boundaries(dims, src_o, *spec_arrays(spec), touches)
    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.fill_periodic(periodic, full=True)
    blk.apply_boundaries(spec, touches)
    blk.sync()
    got = blk.download_src()
    assert n_bit_mismatch(got, src_o) == 0


def test_device_observers_match_sample_scalars(gpu, oracle):
    """lbg_observe == the fluid part of io::sample_scalars (output.cpp:22-45): mass and bare
    momentum as total_mass/total_momentum (lbm.cpp:69-93), KE with the half-force-shifted
    velocity; compensated device reduction, relative 1e-14 of the oracle's serial sums."""
    dims = (40, 33, 27)
    src = random_pdf(dims, seed=55)
    fext = (2e-5, -1e-5, 3e-6)
    blk = gpu.Block(dims)
    blk.upload_src(src)
    obs = blk.observe(fext)
    mass = oracle.total_mass(dims, src)
    mom = oracle.total_momentum(dims, src)
    f = interior(src)
    cxyz = np.array([[0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0],
                     [0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1],
                     [0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1]], float)
    rho = f.sum(axis=0)
    u = np.einsum("aq,qkji->akji", cxyz, f) + 0.5 * np.array(fext)[:, None, None, None]
    u2 = (u * u).sum(axis=0)
    ke = float(np.sum(0.5 * rho * u2, dtype=np.float64))
    assert abs(obs["mass"] - mass) <= 1e-14 * abs(mass)
    assert np.all(np.abs(obs["momentum"] - mom) <= 1e-13 * np.abs(f).sum())
    assert abs(obs["fluid_ke"] - ke) <= 1e-12 * ke
    assert abs(obs["max_u"] - np.sqrt(u2.max())) <= 1e-15
    assert abs(blk.total_mass() - mass) <= 1e-14 * mass


@pytest.mark.parametrize("coupled,dims", [(False, (37, 21, 19)), (True, (37, 21, 19)),
                                          (True, (150, 131, 120))])
def test_device_moments_bitwise(gpu, oracle, coupled, dims):
    """lbg_moments: per-cell {rho, mx, my, mz[, btot]} equal to the reference's per-cell sums
    (lbm.cpp:61-93) bit for bit, so observers and grid dumps built on the host from 32-40 B
    per cell reproduce total_mass / total_momentum / write_grid_dump exactly. The large case
    crosses the 64 MB z-chunk staging (two chunks)."""
    src = random_pdf(dims, seed=77)
    blk = gpu.Block(dims, coupling=coupled)
    blk.upload_src(src)
    want = oracle.moments(dims, src)
    if coupled:
        frac, _ = random_fraction(dims, seed=8)
        blk.upload_fraction(frac)
    got = blk.moments(with_frac=True)
    assert n_bit_mismatch(got[..., :4], want) == 0
    btot = frac["btot"].reshape(dims[::-1]) if coupled else np.zeros(dims[::-1])
    assert equal_bits(got[..., 4], btot)
    assert n_bit_mismatch(blk.moments(with_frac=False), want) == 0


def test_pinned_chunked_transfers_roundtrip(gpu):
    """Large PDF transfers from/to pinned host memory take the chunked linear-copy + re-pitch
    path; they must round-trip exactly and agree with the pageable 2-D copy path."""
    import ctypes as C
    from paper_2303_11811_b200 import lbg as abi
    dims = (150, 131, 120)  # 19 * 152 * 133 * 122 * 8 B = 375 MB > 64 MB threshold
    shape = (19, dims[2] + 2, dims[1] + 2, dims[0] + 2)
    nbytes = 8 * int(np.prod(shape))
    hp = C.c_void_p()
    gpu.check(abi.load().lbg_host_alloc(nbytes, C.byref(hp)))
    try:
        pinned = np.ctypeslib.as_array(C.cast(hp, C.POINTER(C.c_double)), shape=shape)
        rng = np.random.default_rng(3)
        pinned[...] = rng.random(shape)
        ref = pinned.copy()
        blk = gpu.Block(dims)
        gpu.check(abi.load().lbg_upload_src(blk.h, hp))
        assert equal_bits(blk.download_src(), ref)  # pageable download (2-D copy path)
        pinned[...] = 0.0
        gpu.check(abi.load().lbg_download_src(blk.h, hp))  # pinned download (chunked path)
        assert equal_bits(pinned, ref)
    finally:
        abi.load().lbg_host_free(hp)


def test_stability_guard_raises(gpu):
    dims = (4, 4, 4)
    blk = gpu.Block(dims)
    blk.fill_equilibrium(1.0, (0.0, 0.0, 0.0))
    a = blk.download_src()
    a[1, 3, 3, 3] = 5.0  # test_lattice_lbm.cpp:324-334
    blk.upload_src(a)
    gpu.fill_periodic_ghosts(blk, ALL_P)
    with pytest.raises(gpu.NumericError, match="fluid instability"):
        gpu.collide_stream(blk, gpu.FluidParams(0.51), gpu.CellBox((0, 0, 0), dims))


@pytest.mark.parametrize("coupled", [False, True])
def test_unstable_cell_count_matches_reference(gpu, oracle, coupled):
    """lbm.cpp:47-48 / psm.cpp:260-261: the NumericError message carries the number of unstable
    cells; the device ballot count (K1 fluid warps, K2 fluid and covered lanes, the shell)
    equals the oracle's count, cells scattered over row segments of both kinds."""
    import re
    dims = (70, 9, 6)
    src0 = random_pdf(dims, seed=123)
    rng = np.random.default_rng(5)
    inner = interior(src0)
    for _ in range(37):  # push |u|^2 past 0.57^2 in scattered cells
        i, j, k = rng.integers(0, dims[0]), rng.integers(0, dims[1]), rng.integers(0, dims[2])
        inner[1, k, j, i] = 2.0
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    tau, fext = 0.7, (0.0, 0.0, 0.0)
    blk = gpu.Block(dims, coupling=coupled)
    if coupled:
        frac, sv = random_fraction(dims, seed=6, cover=0.3)
        scr = new_scratch(dims)
        bad = oracle.psm_collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims, frac, sv, scr)
        blk.upload_fraction(frac)
        blk.upload_solid_velocity(sv["v0"], sv["v1"])
    else:
        bad = oracle.collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims)
    assert 10 < bad <= 37
    blk.upload_src(src0)
    blk.fill_periodic(ALL_P, full=True)
    blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox((0, 0, 0), dims))
    with pytest.raises(gpu.NumericError) as e:
        blk.sync()
    assert int(re.search(r"instability[^:]*: (\d+)", str(e.value)).group(1)) == bad


def test_config_validation_errors(gpu):
    blk = gpu.Block((4, 4, 4))
    with pytest.raises(gpu.ConfigError):
        blk.sweep(gpu.FluidParams(0.4), gpu.CellBox((0, 0, 0), (4, 4, 4)))
    spec = gpu.BcSpec()
    spec.faces[2] = gpu.FaceBc(gpu.BcKind.no_slip)
    with pytest.raises(gpu.ConfigError):
        blk.apply_boundaries(spec, (1,) * 6)


def shear_wave(oracle, dims):
    nx, ny, nz = dims
    a = np.zeros((19, nz + 2, ny + 2, nx + 2))
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                u = (0.02 * np.sin(2.0 * np.pi * (j + 0.5) / ny), 0.015 * np.cos(2.0 * np.pi * (k + 0.5) / nz),
                     0.01 * np.sin(2.0 * np.pi * (i + 0.5) / nx))
                a[:, k + 1, j + 1, i + 1] = oracle.equilibrium(1.0, u)
    return a


def test_shear_wave_100_steps_bitwise(gpu, oracle):
    """SURVEY.md §7 minimum slice: periodic shear wave, tau 0.8, 1 and 100 steps."""
    dims = (24, 20, 16)
    src = shear_wave(oracle, dims)
    blk = gpu.Block(dims)
    blk.upload_src(src)
    p = gpu.FluidParams(0.8)
    o_src = src.copy()
    for step in range(100):
        dst = np.zeros_like(o_src)
        oracle.fill_periodic(dims, o_src, ALL_P)
        oracle.collide_stream(dims, o_src, dst, 0.8, (0, 0, 0), (0, 0, 0), dims)
        o_src = dst
        blk.fill_periodic(ALL_P, full=False)
        blk.sweep(p, gpu.CellBox((0, 0, 0), dims))
        blk.swap()
        if step in (0, 99):
            blk.sync()
            assert equal_bits(interior(blk.download_src()), interior(o_src)), f"step {step + 1}"
    m = blk.total_mass()
    assert abs(m - oracle.total_mass(dims, o_src)) <= 1e-12 * m


# ----------------------------------------------------------------------------- PSM
def random_fraction(dims, seed, n_ids=4, cover=0.4):
    rng = np.random.default_rng(seed)
    nx, ny, nz = dims
    f = new_fraction(dims)
    cnt = rng.random((nz, ny, nx))
    f["count"][:] = np.where(cnt < cover / 2, 2, np.where(cnt < cover, 1, 0)).astype(np.uint8)
    f["id0"][:] = rng.integers(0, n_ids, (nz, ny, nx))
    f["id1"][:] = rng.integers(0, n_ids, (nz, ny, nx))
    f["b0"][:] = rng.random((nz, ny, nx))
    f["b1"][:] = rng.random((nz, ny, nx)) * (1 - f["b0"])
    f["btot"][:] = np.minimum(1.0, f["b0"] + np.where(f["count"] > 1, f["b1"], 0.0))
    sv = new_svel(dims)
    sv["v0"][:] = 0.02 * (rng.random((nz, ny, nx, 3)) - 0.5)
    sv["v1"][:] = 0.02 * (rng.random((nz, ny, nx, 3)) - 0.5)
    return f, sv


@pytest.mark.parametrize("fext", [(0.0, 0.0, 0.0), (1e-5, 0.0, -4e-6)])
def test_psm_sweep_bitwise(gpu, oracle, fext):
    dims = (12, 10, 9)
    src0 = random_pdf(dims, seed=67)
    frac, sv = random_fraction(dims, seed=1)
    tau = 0.65
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    scr = new_scratch(dims)
    bad = oracle.psm_collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims, frac, sv, scr)
    assert bad == 0
    blk = gpu.Block(dims, coupling=True)
    blk.upload_src(src0)
    blk.upload_fraction(frac)
    blk.upload_solid_velocity(sv["v0"], sv["v1"])
    blk.fill_periodic(ALL_P, full=True)
    blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox((0, 0, 0), dims))
    blk.sync()
    assert n_bit_mismatch(interior(blk.download_dst()), interior(dst_o)) == 0
    m0, m1 = blk.download_scratch()
    c = frac["count"]
    assert equal_bits(m0[c > 0], scr["m0"][c > 0])
    assert equal_bits(m1[c > 1], scr["m1"][c > 1])


@pytest.mark.parametrize("fext", [(0.0, 0.0, 0.0), (0.0, 2e-6, 0.0)])
@pytest.mark.parametrize("cover", [0.05, 0.4, 0.9])
def test_psm_one_entry_segments_bitwise(gpu, oracle, fext, cover):
    """K2's one-entry segments (no two-entry cell): fluid and covered lanes of one warp share
    the one-entry operator when unforced (B = b = 0, v = 0 is collide_cell exactly) and take
    SRT / PSM in turn when forced — bitwise either way, sparse to dense cover, long rows."""
    dims = (70, 6, 5)
    src0 = random_pdf(dims, seed=91)
    frac, sv = random_fraction(dims, seed=13, cover=cover)
    frac["count"][:] = np.minimum(frac["count"], 1)
    frac["btot"][:] = np.minimum(1.0, frac["b0"])
    tau = 0.6
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    scr = new_scratch(dims)
    assert oracle.psm_collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims, frac, sv, scr) == 0
    blk = gpu.Block(dims, coupling=True)
    blk.upload_src(src0)
    blk.upload_fraction(frac)
    blk.upload_solid_velocity(sv["v0"], sv["v1"])
    blk.fill_periodic(ALL_P, full=True)
    blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox((0, 0, 0), dims))
    blk.sync()
    assert n_bit_mismatch(interior(blk.download_dst()), interior(dst_o)) == 0
    m0, _ = blk.download_scratch()
    c = frac["count"]
    assert equal_bits(m0[c > 0], scr["m0"][c > 0])


def test_psm_with_zero_fraction_is_plain_srt(gpu, oracle):
    """test_psm.cpp:269-304 — B = 0 PSM == SRT, bitwise."""
    dims = (12, 12, 12)
    src0 = random_pdf(dims, seed=68)
    p = gpu.FluidParams(0.8, (1e-5, 0.0, 0.0))
    a = gpu.Block(dims, coupling=True)
    b = gpu.Block(dims)
    for blk in (a, b):
        blk.upload_src(src0)
        blk.fill_periodic(ALL_P)
        blk.sweep(p, gpu.CellBox((0, 0, 0), dims))
        blk.sync()
    assert equal_bits(a.download_dst(), b.download_dst())


def spheres(oracle, centers, radii, ids=None, u=None, w=None):
    n = len(centers)
    ids = list(range(n)) if ids is None else ids
    fr = [oracle.f_of_r(r) for r in radii]
    return make_snapshots(ids, centers, radii, fr, u, w)


@pytest.mark.parametrize("lo", [(0, 0, 0), (16, 8, 24)])
def test_mapping_and_solid_velocity_bitwise(gpu, oracle, lo):
    dims = (40, 36, 44)
    rng = np.random.default_rng(7)
    centers = [(lo[0] + 10.3, lo[1] + 12.6, lo[2] + 11.2), (lo[0] + 19.0, lo[1] + 12.1, lo[2] + 12.0),
               (lo[0] + 28.4, lo[1] + 25.5, lo[2] + 30.1), (lo[0] + 1.0, lo[1] + 30.0, lo[2] + 40.5),
               (lo[0] - 3.0, lo[1] + 2.0, lo[2] + 2.0)]  # last one is a ghost poking in
    radii = [6.0, 5.0, 8.5, 4.0, 5.5]
    u = 0.01 * (rng.random((5, 3)) - 0.5)
    w = 0.002 * (rng.random((5, 3)) - 0.5)
    s = spheres(oracle, centers, radii, ids=[2, 5, 9, 11, 40], u=u, w=w)
    f_o, over = oracle.build_fraction_field(lo, dims, s)
    assert over == 0
    sv_o, unk = oracle.set_solid_velocities(lo, dims, s, f_o)
    assert unk == 0
    blk = gpu.Block(dims, lo=lo, coupling=True)
    gpu.build_fraction_field(blk, s)
    f = blk.download_fraction()
    c = f["count"]
    assert np.array_equal(c, f_o["count"])
    assert (c == 2).any()
    assert equal_bits(f["btot"], f_o["btot"])
    for e, (idk, bk, vk) in enumerate((("id0", "b0", "v0"), ("id1", "b1", "v1"))):
        sel = c > e
        assert np.array_equal(f[idk][sel], f_o[idk][sel])
        assert equal_bits(f[bk][sel], f_o[bk][sel])
    v0, v1 = blk.download_solid_velocity()
    assert equal_bits(v0[c > 0], sv_o["v0"][c > 0])
    assert equal_bits(v1[c > 1], sv_o["v1"][c > 1])


@pytest.mark.parametrize("id_step", [1, 1000])
def test_mapping_dense_bins_bitwise(gpu, oracle, id_step):
    """2197 small spheres (r = 0.75) on a jittered 1.8-cell lattice: ~125 candidates per 8^3
    bin, so the bin-major mapping kernel stages them in several shared-memory chunks; 1662
    two-entry cells. Fraction field, ids and solid velocities bitwise vs build_fraction_field /
    set_solid_velocities. Dense ids use the id -> index table, sparse ids (step 1000) the
    binary search."""
    dims = (24, 24, 24)
    rng = np.random.default_rng(3)
    g = np.arange(1.2, 24, 1.8)
    centers = np.array([(x, y, z) for z in g for y in g for x in g]) + (rng.random((len(g) ** 3, 3)) - 0.5) * 0.2
    n = len(centers)
    s = spheres(oracle, centers, [0.75] * n, ids=[id_step * i for i in range(n)],
                u=0.01 * (rng.random((n, 3)) - 0.5), w=0.002 * (rng.random((n, 3)) - 0.5))
    f_o, over = oracle.build_fraction_field((0, 0, 0), dims, s)
    assert over == 0
    sv_o, _ = oracle.set_solid_velocities((0, 0, 0), dims, s, f_o)
    blk = gpu.Block(dims, coupling=True)
    gpu.build_fraction_field(blk, s)
    gpu.set_solid_velocities(blk, s)
    f = blk.download_fraction()
    c = f["count"]
    assert np.array_equal(c, f_o["count"]) and (c == 2).sum() > 1000
    assert equal_bits(f["btot"], f_o["btot"])
    for e, (idk, bk, vk) in enumerate((("id0", "b0", "v0"), ("id1", "b1", "v1"))):
        sel = c > e
        assert np.array_equal(f[idk][sel], f_o[idk][sel])
        assert equal_bits(f[bk][sel], f_o[bk][sel])
    v0, v1 = blk.download_solid_velocity()
    assert equal_bits(v0[c > 0], sv_o["v0"][c > 0])
    assert equal_bits(v1[c > 1], sv_o["v1"][c > 1])


def test_mapping_dense_bins_overfull_raises(gpu, oracle):
    """The same lattice at 1.6-cell spacing has cells inside three spheres (77 of them)."""
    g = np.arange(1.2, 24, 1.6)
    centers = np.array([(x, y, z) for z in g for y in g for x in g]) + \
        (np.random.default_rng(3).random((len(g) ** 3, 3)) - 0.5) * 0.2
    s = spheres(oracle, centers, [0.75] * len(centers))
    assert oracle.build_fraction_field((0, 0, 0), (24, 24, 24), s)[1] == 77
    blk = gpu.Block((24, 24, 24), coupling=True)
    with pytest.raises(gpu.NumericError, match="more than two particles"):
        gpu.build_fraction_field(blk, s)


def test_mapping_overfull_raises(gpu, oracle):
    """test_psm.cpp:166-176 — three particles through one cell."""
    dims = (40, 40, 40)
    s = spheres(oracle, [(20.0 + 0.4 * i, 20.0, 20.0) for i in range(3)], [10.0] * 3)
    blk = gpu.Block(dims, coupling=True)
    with pytest.raises(gpu.NumericError, match="more than two particles"):
        gpu.build_fraction_field(blk, s)


def test_set_solid_velocities_unknown_id(gpu, oracle):
    """test_psm.cpp:414-424."""
    dims = (16, 16, 16)
    f = new_fraction(dims)
    f["count"][8, 8, 8] = 1
    f["id0"][8, 8, 8] = 42
    f["b0"][8, 8, 8] = 0.5
    blk = gpu.Block(dims, coupling=True)
    blk.upload_fraction(f)
    with pytest.raises(gpu.SyncError, match="unknown particle ids"):
        gpu.set_solid_velocities(blk, make_snapshots([], np.zeros((0, 3)), [], []))


def _moved(oracle, s, rng):
    """The post-sync snapshot list: same particles, new velocities, plus a ghost id the
    mapping never saw (sim.cpp:249-267 refreshes u and omega between mapping and setU)."""
    n = len(s["id"])
    return make_snapshots(list(s["id"]) + [int(max(s["id"])) + 7], list(s["x"]) + [(500.0, 500.0, 500.0)],
                          list(s["r"]) + [3.0], list(s["f_r"]) + [oracle.f_of_r(3.0)],
                          list(0.01 * (rng.random((n, 3)) - 0.5)) + [(0.0, 0.0, 0.0)],
                          list(0.002 * (rng.random((n, 3)) - 0.5)) + [(0.0, 0.0, 0.0)])


@pytest.mark.parametrize("fused", [False, True])
def test_setu_after_velocity_sync_inline_bitwise(gpu, oracle, fused):
    """map(A) -> set_solid_velocities(B: new u/omega, one extra id) -> PSM sweep: the PSM
    kernels evaluate u + omega x (c - x) from B inline (no v0/v1 traffic); PDFs, scratch and
    the downloaded (materialised) solid velocities are bitwise the reference's setU(B)."""
    dims = (32, 30, 34)
    src0 = random_pdf(dims, seed=93)
    rng = np.random.default_rng(21)
    centers = [(9.2, 10.1, 11.7), (17.5, 10.4, 12.2), (22.0, 21.0, 23.3), (8.0, 24.0, 26.0)]
    a = spheres(oracle, centers, [5.0, 4.5, 6.0, 3.5], ids=[1, 3, 4, 8],
                u=0.01 * (rng.random((4, 3)) - 0.5), w=0.001 * (rng.random((4, 3)) - 0.5))
    b = _moved(oracle, a, rng)
    tau, fext = 0.7, (0.0, 0.0, -1e-5)
    f_o, _ = oracle.build_fraction_field((0, 0, 0), dims, a)
    sv_o, unk = oracle.set_solid_velocities((0, 0, 0), dims, b, f_o)
    assert unk == 0 and (f_o["count"] == 2).any()
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    scr = new_scratch(dims)
    oracle.psm_collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims, f_o, sv_o, scr)
    blk = gpu.Block(dims, coupling=True)
    if fused:
        blk.set_force_mode(1)
    blk.upload_src(src0)
    gpu.build_fraction_field(blk, a)
    gpu.set_solid_velocities(blk, b)
    blk.fill_periodic(ALL_P)
    p = gpu.FluidParams(tau, fext)
    blk.sweep(p, gpu.CellBox((1, 1, 1), (dims[0] - 1, dims[1] - 1, dims[2] - 1)))
    blk.sweep_boxes(p, gpu.boundary_shell(dims))  # shell cells: the flat coupled kernel
    blk.sync()
    assert equal_bits(interior(blk.download_dst()), interior(dst_o))
    c = f_o["count"]
    if not fused:
        m0, m1 = blk.download_scratch()
        assert equal_bits(m0[c > 0], scr["m0"][c > 0]) and equal_bits(m1[c > 1], scr["m1"][c > 1])
    v0, v1 = blk.download_solid_velocity()
    assert equal_bits(v0[c > 0], sv_o["v0"][c > 0])
    assert equal_bits(v1[c > 1], sv_o["v1"][c > 1])


def test_setu_missing_mapped_id_raises(gpu, oracle):
    """A post-sync list that lost a particle the field still names: SyncError from
    set_solid_velocities, as psm.cpp:165-168 (the exact per-entry walk runs then)."""
    dims = (24, 24, 24)
    a = spheres(oracle, [(8.0, 8.0, 8.0), (16.0, 16.0, 16.0)], [4.0, 4.0], ids=[3, 9])
    blk = gpu.Block(dims, coupling=True)
    gpu.build_fraction_field(blk, a)
    b = spheres(oracle, [(8.0, 8.0, 8.0)], [4.0], ids=[3])
    with pytest.raises(gpu.SyncError, match="unknown particle ids"):
        gpu.set_solid_velocities(blk, b)


def test_partial_velocity_upload_keeps_mapped_side(gpu, oracle):
    """Uploading v0 only keeps v1 = the mapped snapshots' setU values (materialised first)."""
    dims = (24, 24, 24)
    rng = np.random.default_rng(5)
    a = spheres(oracle, [(10.0, 12.0, 12.0), (15.5, 12.0, 12.0)], [4.5, 4.5], ids=[0, 1],
                u=0.01 * (rng.random((2, 3)) - 0.5), w=0.002 * (rng.random((2, 3)) - 0.5))
    f_o, _ = oracle.build_fraction_field((0, 0, 0), dims, a)
    sv_o, _ = oracle.set_solid_velocities((0, 0, 0), dims, a, f_o)
    c = f_o["count"]
    assert (c == 2).any()
    blk = gpu.Block(dims, coupling=True)
    gpu.build_fraction_field(blk, a)
    mine = rng.random((24, 24, 24, 3))
    blk.upload_solid_velocity(mine, None)
    v0, v1 = blk.download_solid_velocity()
    assert equal_bits(v0, mine)
    assert equal_bits(v1[c > 1], sv_o["v1"][c > 1])


@pytest.mark.parametrize("mode", [0, 1])
def test_full_coupled_pass_and_reduction(gpu, oracle, mode):
    """map -> setU -> PSM sweep -> finalize: PARITY mode bitwise, FAST within L1 tolerance."""
    dims = (32, 30, 34)
    src0 = random_pdf(dims, seed=90)
    rng = np.random.default_rng(11)
    centers = [(9.2, 10.1, 11.7), (17.5, 10.4, 12.2), (22.0, 21.0, 23.3), (8.0, 24.0, 26.0)]
    s = spheres(oracle, centers, [5.0, 4.5, 6.0, 3.5], ids=[1, 3, 4, 8],
                u=0.01 * (rng.random((4, 3)) - 0.5), w=0.001 * (rng.random((4, 3)) - 0.5))
    tau, fext = 0.7, (0.0, 0.0, -1e-5)
    f_o, _ = oracle.build_fraction_field((0, 0, 0), dims, s)
    sv_o, _ = oracle.set_solid_velocities((0, 0, 0), dims, s, f_o)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    scr = new_scratch(dims)
    oracle.psm_collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims, f_o, sv_o, scr)
    l1 = {}
    for e, mk in ((0, "m0"), (1, "m1")):
        sel = f_o["count"] > e
        ids = f_o["id0" if e == 0 else "id1"][sel]
        for pid, mv in zip(ids, np.abs(scr[mk][sel])):
            l1[int(pid)] = l1.get(int(pid), 0) + mv
    ids_o, rows_o = oracle.finalize_hydro((0, 0, 0), dims, s, f_o, scr)

    blk = gpu.Block(dims, coupling=True)
    blk.upload_src(src0)
    blk.map(s)
    blk.fill_periodic(ALL_P)
    blk.sweep(gpu.FluidParams(tau, fext), gpu.CellBox((0, 0, 0), dims))
    blk.sync()
    assert equal_bits(interior(blk.download_dst()), interior(dst_o))
    parts = gpu.finalize_hydro_forces(blk, mode)
    assert [p.id for p in parts] == list(ids_o)
    for p, r in zip(parts, rows_o):
        if mode == 0:
            assert equal_bits(np.concatenate([p.f, p.f_comp, p.t, p.t_comp]), r)
        else:
            assert np.all(np.abs((p.f + p.f_comp) - (r[0:3] + r[3:6])) <= 1e-12 * l1[p.id] + 1e-300)
    m0, m1 = blk.download_scratch()
    assert not m0.any() and not m1.any()  # finalize clears the scratch


def test_fused_force_mode_within_l1_tolerance(gpu, oracle):
    """LBG_FORCE_FUSED: force/torque summed inside the PSM kernel (warp aggregation by particle
    + atomics); PDFs stay bitwise, partials within |dF| <= 1e-12 * sum|m| (and the same for
    the torque with sum |r x m|)."""
    dims = (32, 30, 34)
    src0 = random_pdf(dims, seed=91)
    rng = np.random.default_rng(12)
    centers = [(9.2, 10.1, 11.7), (17.5, 10.4, 12.2), (22.0, 21.0, 23.3), (8.0, 24.0, 26.0)]
    s = spheres(oracle, centers, [5.0, 4.5, 6.0, 3.5], ids=[1, 3, 4, 8],
                u=0.01 * (rng.random((4, 3)) - 0.5), w=0.001 * (rng.random((4, 3)) - 0.5))
    tau, fext = 0.7, (0.0, 0.0, -1e-5)
    f_o, _ = oracle.build_fraction_field((0, 0, 0), dims, s)
    sv_o, _ = oracle.set_solid_velocities((0, 0, 0), dims, s, f_o)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    scr = new_scratch(dims)
    oracle.psm_collide_stream(dims, src_o, dst_o, tau, fext, (0, 0, 0), dims, f_o, sv_o, scr)
    l1f, l1t = {}, {}
    for e, mk in ((0, "m0"), (1, "m1")):
        sel = f_o["count"] > e
        ids = f_o["id0" if e == 0 else "id1"][sel]
        kk, jj, ii = np.nonzero(sel)
        for pid, mv, i, j, k in zip(ids, scr[mk][sel], ii, jj, kk):
            x = s["x"][list(s["id"]).index(pid)]
            r = np.array([i + 0.5, j + 0.5, k + 0.5]) - x
            l1f[int(pid)] = l1f.get(int(pid), 0) + np.abs(mv)
            l1t[int(pid)] = l1t.get(int(pid), 0) + np.abs(np.cross(r, mv))
    ids_o, rows_o = oracle.finalize_hydro((0, 0, 0), dims, s, f_o, scr)
    blk = gpu.Block(dims, coupling=True)
    blk.set_force_mode(1)
    blk.upload_src(src0)
    blk.map(s)
    blk.fill_periodic(ALL_P)
    p = gpu.FluidParams(tau, fext)
    blk.sweep(p, gpu.CellBox((1, 1, 1), (dims[0] - 1, dims[1] - 1, dims[2] - 1)))
    blk.sweep_boxes(p, gpu.boundary_shell(dims))  # two launches accumulate into one sum
    blk.sync()
    assert equal_bits(interior(blk.download_dst()), interior(dst_o))
    with pytest.raises(ValueError):
        gpu.finalize_hydro_forces(blk, 0)  # PARITY needs the scratch
    parts = gpu.finalize_hydro_forces(blk, 1)
    assert [q.id for q in parts] == list(ids_o)
    for q, r in zip(parts, rows_o):
        assert np.all(np.abs(q.f - (r[0:3] + r[3:6])) <= 1e-12 * l1f[q.id])
        assert np.all(np.abs(q.t - (r[6:9] + r[9:12])) <= 1e-12 * l1t[q.id] + 1e-300)


def test_finalize_symmetric_pattern(gpu, oracle):
    """test_psm.cpp:386-412: no cover -> no partials; symmetric pattern -> 6*0.01, zero torque."""
    dims = (16, 16, 16)
    s = spheres(oracle, [(8.5, 8.5, 8.5)], [3.0])
    blk = gpu.Block(dims, coupling=True)
    blk.map(make_snapshots([0], [(100.0, 100.0, 100.0)], [3.0], [oracle.f_of_r(3.0)]))
    blk.sync()
    blk.set_solid_velocities(s)  # registers the snapshot list used by the reduction
    blk.sync()
    assert gpu.finalize_hydro_forces(blk) == []
    f = new_fraction(dims)
    m0 = np.zeros((16, 16, 16, 3))
    for c in [(6, 8, 8), (10, 8, 8), (8, 6, 8), (8, 10, 8), (8, 8, 6), (8, 8, 10)]:
        i, j, k = c
        f["count"][k, j, i] = 1
        f["id0"][k, j, i] = 0
        f["b0"][k, j, i] = 0.5
        m0[k, j, i] = (0.01, 0.0, 0.0)
    blk.upload_fraction(f)
    blk.upload_scratch(m0, np.zeros_like(m0))
    parts = gpu.finalize_hydro_forces(blk)
    assert len(parts) == 1
    assert abs(parts[0].f[0] - 0.06) <= 1e-13 * 0.06
    assert np.linalg.norm(parts[0].t + parts[0].t_comp) < 1e-14


def test_single_rank_halo_equals_periodic_fill(gpu, oracle):
    """K7 with one rank and a periodic z axis is the local z wrap of the ghost planes."""
    dims = (10, 8, 6)
    src0 = random_pdf(dims, seed=12)
    tau = 0.8
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    oracle.collide_stream(dims, src_o, dst_o, tau, (0, 0, 0), (0, 0, 0), dims)
    blk = gpu.Block(dims)
    blk.comm_init(1, 0, b"\0" * 128, axis=2, periodic=ALL_P)
    blk.upload_src(src0)
    blk.fill_periodic((1, 1, 0), full=False)
    blk.halo_begin()
    p = gpu.FluidParams(tau)
    blk.sweep(p, gpu.CellBox((0, 0, 1), (dims[0], dims[1], dims[2] - 1)))
    blk.halo_complete()
    blk.sweep_boxes(p, [gpu.CellBox((0, 0, 0), (dims[0], dims[1], 1)),
                        gpu.CellBox((0, 0, dims[2] - 1), dims)])
    blk.sync()
    assert equal_bits(interior(blk.download_dst()), interior(dst_o))
    with pytest.raises(gpu.SyncError):
        blk.halo_complete()
    # the bench's weak-scaling step shape: x/y wrapped in-kernel, z through the halo
    blk2 = gpu.Block(dims)
    blk2.comm_init(1, 0, b"\0" * 128, axis=2, periodic=ALL_P)
    blk2.upload_src(src0)
    blk2.set_periodic_wrap((1, 1, 0))
    blk2.halo_begin()
    blk2.sweep(p, gpu.CellBox((0, 0, 1), (dims[0], dims[1], dims[2] - 1)))
    blk2.halo_complete()
    blk2.sweep_boxes(p, [gpu.CellBox((0, 0, 0), (dims[0], dims[1], 1)),
                         gpu.CellBox((0, 0, dims[2] - 1), dims)])
    blk2.sync()
    assert equal_bits(interior(blk2.download_dst()), interior(dst_o))


@pytest.mark.parametrize("grid,batched", [((1, 1, 1), False), ((2, 2, 1), False), ((2, 2, 1), True)])
def test_poisoned_halos_never_leak(gpu, oracle, grid, batched):
    """test_partition.cpp:130-151 on the device path: every block's ghosts are NaN, the
    26-neighbour halo runs device to device (lbg_halo_stage / lbg_halo_fetch, periodic
    self-messages included), then a full sweep. Every interior population is finite and the
    decomposed step equals the single-domain oracle step bitwise (test_partition.cpp:95-128)."""
    import itertools
    D = (12, 12, 12)
    tau, fext = 0.8, (1e-6, 0.0, 0.0)
    bd = tuple(D[a] // grid[a] for a in range(3))
    offs = [o for o in itertools.product((-1, 0, 1), repeat=3) if any(o)]
    src_g = random_pdf(D, seed=101)
    blocks = {}
    for g in itertools.product(*(range(n) for n in grid)):
        lo = tuple(g[a] * bd[a] for a in range(3))
        b = gpu.Block(bd, lo=lo)
        sub = np.full((19, bd[2] + 2, bd[1] + 2, bd[0] + 2), np.nan)
        sub[:, 1:-1, 1:-1, 1:-1] = interior(src_g)[:, lo[2]:lo[2] + bd[2], lo[1]:lo[1] + bd[1],
                                                    lo[0]:lo[0] + bd[0]]
        b.upload_src(sub)
        b.fill_ghosts_src(np.nan)
        blocks[g] = b
    for b in blocks.values():
        b.halo_stage(offs)
    for g, b in blocks.items():
        entries = [(o, blocks[tuple((g[a] + o[a]) % grid[a] for a in range(3))]) for o in offs]
        if batched:  # lbg_halo_fetch_all: every neighbour entry in one unpack launch
            b.halo_fetch_all(entries)
        else:
            for o, nb in entries:
                b.halo_fetch(o, nb)
    p = gpu.FluidParams(tau, fext)
    for b in blocks.values():
        b.sweep(p, gpu.CellBox((0, 0, 0), bd))
        b.sync()
    src_o = src_g.copy()
    oracle.fill_periodic(D, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    oracle.collide_stream(D, src_o, dst_o, tau, fext, (0, 0, 0), D)
    want = interior(dst_o)
    for g, b in blocks.items():
        lo = tuple(g[a] * bd[a] for a in range(3))
        got = interior(b.download_dst())
        assert np.isfinite(got).all()
        assert n_bit_mismatch(got, want[:, lo[2]:lo[2] + bd[2], lo[1]:lo[1] + bd[1], lo[0]:lo[0] + bd[0]]) == 0


def test_fused_mode_switched_after_map_with_longer_setu_list(gpu, oracle):
    """The fused accumulators follow the force mode and the snapshot list (advisor findings):
    the mode is switched to FUSED after the mapping, and set_solid_velocities then registers a
    LONGER list than the mapping's (two extra ghost ids). The accumulators must cover the longer
    list (sized and zeroed by set_solid_velocities), the sweep must not run without them, and
    the FAST partials match the oracle's walk over the same list within the L1 tolerance."""
    dims = (24, 22, 26)
    src0 = random_pdf(dims, seed=95)
    s_map = spheres(oracle, [(8.2, 9.1, 10.7), (15.5, 11.4, 13.2)], [4.5, 4.0], ids=[2, 5])
    s_all = spheres(oracle, [(8.2, 9.1, 10.7), (15.5, 11.4, 13.2), (60.0, 60.0, 60.0), (70.0, 2.0, 3.0)],
                    [4.5, 4.0, 3.0, 3.0], ids=[2, 5, 9, 11],
                    u=[(0.001, 0.0, -0.002), (0.0, 0.003, 0.0), (0, 0, 0), (0, 0, 0)],
                    w=[(0.0, 0.0005, 0.0), (0.0002, 0.0, 0.0), (0, 0, 0), (0, 0, 0)])
    tau = 0.75
    f_o, _ = oracle.build_fraction_field((0, 0, 0), dims, s_map)
    sv_o, _ = oracle.set_solid_velocities((0, 0, 0), dims, s_all, f_o)
    src_o = src0.copy()
    oracle.fill_periodic(dims, src_o, ALL_P)
    dst_o = np.zeros_like(src_o)
    scr = new_scratch(dims)
    oracle.psm_collide_stream(dims, src_o, dst_o, tau, (0.0, 0.0, 0.0), (0, 0, 0), dims, f_o, sv_o, scr)
    l1 = {}  # before the finalize walk, which clears the scratch (psm.cpp:305)
    for e, mk in ((0, "m0"), (1, "m1")):
        sel = f_o["count"] > e
        for pid, mv in zip(f_o["id0" if e == 0 else "id1"][sel], scr[mk][sel]):
            l1[int(pid)] = l1.get(int(pid), 0) + np.abs(mv)
    ids_o, rows_o = oracle.finalize_hydro((0, 0, 0), dims, s_all, f_o, scr)
    blk = gpu.Block(dims, coupling=True)
    blk.upload_src(src0)
    blk.map(s_map)          # scratch mode: no accumulators yet
    blk.set_force_mode(1)   # takes effect at once: accumulators for the mapping's list
    blk.set_solid_velocities(s_all)  # a longer list: accumulators resized and zeroed
    blk.fill_periodic(ALL_P)
    blk.sweep(gpu.FluidParams(tau), gpu.CellBox((0, 0, 0), dims))
    blk.sync()
    assert equal_bits(interior(blk.download_dst()), interior(dst_o))
    parts = gpu.finalize_hydro_forces(blk, 1)
    assert [q.id for q in parts] == list(ids_o)
    for q, r in zip(parts, rows_o):
        assert np.all(np.abs(q.f - (r[0:3] + r[3:6])) <= 1e-12 * l1[q.id])
