"""The reference's own unit tests for the GPU-side operators, re-run on the CUDA path
(test_lattice_lbm.cpp, test_psm.cpp, test_boundary.cpp; file:line in each docstring). The
parity files prove bitwise equality with the oracle; these keep the reference's physical
expectations visible on the product path."""
import numpy as np
import pytest

from conftest import W, equal_bits, interior, random_pdf
from oracle.pyoracle import make_snapshots, new_fraction, new_svel

pytestmark = pytest.mark.gpu
ALL_P = (1, 1, 1)


def step(gpu, blk, params, periodic=ALL_P):
    blk.fill_periodic(periodic, full=True)
    gpu.collide_stream(blk, params, gpu.CellBox((0, 0, 0), blk.dims))
    blk.swap()


def test_stream_moves_single_population(gpu):
    """test_lattice_lbm.cpp:175-189."""
    dims = (6, 6, 6)
    a = np.zeros((19, 8, 8, 8))
    a[7, 3, 3, 3] = 1.0  # q = 7 (1,1,0) at (2,2,2)
    blk = gpu.Block(dims)
    blk.upload_src(a)
    blk.fill_periodic(ALL_P)
    blk.stream_only(gpu.CellBox((0, 0, 0), dims))
    out = interior(blk.download_dst())[7]
    want = np.zeros((6, 6, 6))
    want[2, 3, 3] = 1.0  # (k, j, i) = (2, 3, 3)
    assert np.array_equal(out, want)


def test_mass_conservation_1000_steps(gpu):
    """test_lattice_lbm.cpp:303-322: periodic force-free domain, 1000 steps, |dm| < 1e-10."""
    dims = (8, 8, 8)
    f = np.zeros((19, 10, 10, 10))
    from oracle.pyoracle import Oracle
    orc = Oracle()
    for k in range(8):
        for j in range(8):
            for i in range(8):
                u = (0.02 * np.sin(2.0 * np.pi * j / 8.0), 0.01 * np.cos(2.0 * np.pi * k / 8.0), 0.0)
                f[:, k + 1, j + 1, i + 1] = orc.equilibrium(1.0, u)
    blk = gpu.Block(dims)
    blk.upload_src(f)
    m0 = orc.total_mass(dims, f)
    blk.set_periodic_wrap(ALL_P)
    p = gpu.FluidParams(0.7)
    for _ in range(1000):
        blk.sweep(p, gpu.CellBox((0, 0, 0), dims))
        blk.swap()
    blk.sync()
    assert abs(orc.total_mass(dims, blk.download_src()) - m0) < 1e-10


def test_no_slip_channel_at_rest_stays_at_rest(gpu):
    """test_boundary.cpp:38-55."""
    dims = (6, 8, 6)
    blk = gpu.Block(dims)
    blk.fill_equilibrium(1.0, (0.0, 0.0, 0.0))
    spec = gpu.BcSpec()
    spec.faces[2] = gpu.FaceBc(gpu.BcKind.no_slip)
    spec.faces[3] = gpu.FaceBc(gpu.BcKind.no_slip)
    blk.fill_periodic((1, 0, 1))
    gpu.apply_boundaries(blk, spec, (1,) * 6)
    gpu.collide_stream(blk, gpu.FluidParams(0.8), gpu.CellBox((0, 0, 0), dims))
    blk.swap()
    out = interior(blk.download_src())
    assert np.all(np.abs(out - W[:, None, None, None]) < 1e-15)


def test_velocity_inflow_injects_rho_u(gpu):
    """test_boundary.cpp:64-94: net mass flux through the inlet plane = rho u_in A."""
    n = 6
    dims = (n, n, 8)
    blk = gpu.Block(dims)
    blk.fill_equilibrium(1.0, (0.0, 0.0, 0.0))
    u_in = 0.01
    spec = gpu.BcSpec()
    spec.faces[4] = gpu.FaceBc(gpu.BcKind.velocity, (0.0, 0.0, u_in))
    spec.faces[5] = gpu.FaceBc(gpu.BcKind.no_slip)
    blk.fill_periodic((1, 1, 0))
    gpu.apply_boundaries(blk, spec, (0, 0, 0, 0, 1, 1))
    f = blk.download_src()
    cz = [0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1]
    cx = [0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0]
    cy = [0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1]
    influx = 0.0
    for j in range(n):
        for i in range(n):
            for q in range(19):
                if cz[q] > 0:  # pulled from ghost k = -1 at (i - cx, j - cy)
                    influx += f[q, 0, j - cy[q] + 1, i - cx[q] + 1]
                elif cz[q] < 0:
                    influx -= f[q, 1, j + 1, i + 1]
    assert abs(influx - u_in * n * n) <= 1e-10 * u_in * n * n


def test_pressure_outflow_relaxes(gpu):
    """test_boundary.cpp:96-115: over-dense channel relaxes to the outlet density."""
    n, nz = 6, 16
    blk = gpu.Block((n, n, nz))
    blk.fill_equilibrium(1.05, (0.0, 0.0, 0.0))
    spec = gpu.BcSpec()
    spec.faces[4] = gpu.FaceBc(gpu.BcKind.no_slip)
    spec.faces[5] = gpu.FaceBc(gpu.BcKind.pressure, (0.0, 0.0, 0.0), 1.0)
    p = gpu.FluidParams(0.8)
    for _ in range(200):
        blk.fill_periodic((1, 1, 0))
        blk.apply_boundaries(spec, (1,) * 6)
        blk.sweep(p, gpu.CellBox((0, 0, 0), (n, n, nz)))
        blk.swap()
    blk.sync()
    rho = interior(blk.download_src())[:, nz - 1, n // 2, n // 2].sum()
    assert abs(rho - 1.0) <= 5e-3


def test_fully_covered_equilibrium_cell_has_no_solid_response(gpu):
    """test_psm.cpp:306-333."""
    dims = (8, 8, 8)
    blk = gpu.Block(dims, coupling=True)
    blk.fill_equilibrium(1.0, (0.0, 0.0, 0.0))
    f = new_fraction(dims)
    f["count"][4, 4, 4] = 1
    f["id0"][4, 4, 4] = 0
    f["b0"][4, 4, 4] = 1.0
    f["btot"][4, 4, 4] = 1.0
    blk.upload_fraction(f)
    sv = new_svel(dims)
    blk.upload_solid_velocity(sv["v0"], sv["v1"])
    blk.fill_periodic(ALL_P)
    gpu.psm_collide_stream(blk, gpu.FluidParams(0.9), gpu.CellBox((0, 0, 0), dims))
    blk.swap()
    m0, _ = blk.download_scratch()
    assert np.linalg.norm(m0[4, 4, 4]) == 0.0
    feq = np.array([0.0] * 19)
    from oracle.pyoracle import Oracle
    feq = Oracle().equilibrium(1.0, (0.0, 0.0, 0.0))
    assert np.array_equal(interior(blk.download_src())[:, 4, 4, 4], feq)


def test_fixed_sphere_in_stream_feels_drag_along_flow(gpu):
    """test_psm.cpp:335-384: drag on a held sphere points along the stream, no side force."""
    from oracle.pyoracle import Oracle
    orc = Oracle()
    n = 32
    blk = gpu.Block((n, n, n), coupling=True)
    blk.fill_equilibrium(1.0, (0.02, 0.0, 0.0))
    s = make_snapshots([0], [(n / 2, n / 2, n / 2)], [6.0], [orc.f_of_r(6.0)])
    gpu.build_fraction_field(blk, s)
    blk.fill_periodic(ALL_P)
    gpu.psm_collide_stream(blk, gpu.FluidParams(0.7), gpu.CellBox((0, 0, 0), (n, n, n)))
    parts = gpu.finalize_hydro_forces(blk)
    assert len(parts) == 1
    assert parts[0].f[0] > 0.0
    assert abs(parts[0].f[1]) < 1e-12 and abs(parts[0].f[2]) < 1e-12


def test_centered_sphere_fraction_volume_within_1pct(gpu):
    """test_psm.cpp:131-141."""
    from oracle.pyoracle import Oracle
    orc = Oracle()
    blk = gpu.Block((40, 40, 40), coupling=True)
    gpu.build_fraction_field(blk, make_snapshots([0], [(20.0, 20.0, 20.0)], [10.0], [orc.f_of_r(10.0)]))
    f = blk.download_fraction()
    vol = f["b0"][f["count"] > 0].sum()
    assert abs(vol - 4.0 / 3.0 * np.pi * 1000.0) / (4.0 / 3.0 * np.pi * 1000.0) < 0.01


def test_no_particles_gives_empty_field_and_no_partials(gpu):
    """test_psm.cpp:120-129 and 386-395."""
    blk = gpu.Block((24, 20, 16), coupling=True)
    gpu.build_fraction_field(blk, make_snapshots([], np.zeros((0, 3)), [], []))
    f = blk.download_fraction()
    assert not f["count"].any() and not f["btot"].any()
    assert gpu.finalize_hydro_forces(blk) == []


def test_tiny_and_degenerate_blocks(gpu, oracle):
    """Blocks thinner than the shell (boundary_shell degenerate case, field.cpp:59-63) and
    odd sizes: inner (empty) + shell sweeps equal the full sweep bitwise."""
    for dims in [(2, 3, 4), (1, 5, 3), (3, 1, 1), (33, 2, 2)]:
        src = random_pdf(dims, seed=sum(dims))
        s = src.copy()
        oracle.fill_periodic(dims, s, ALL_P)
        d = np.zeros_like(s)
        oracle.collide_stream(dims, s, d, 0.8, (1e-6, 0.0, 0.0), (0, 0, 0), dims)
        blk = gpu.Block(dims)
        blk.upload_src(src)
        blk.fill_periodic(ALL_P)
        p = gpu.FluidParams(0.8, (1e-6, 0.0, 0.0))
        blk.sweep(p, gpu.CellBox((1, 1, 1), (dims[0] - 1, dims[1] - 1, dims[2] - 1)))
        blk.sweep_boxes(p, gpu.boundary_shell(dims))
        blk.sync()
        assert equal_bits(interior(blk.download_dst()), interior(d)), dims
