"""Pins the plain-C oracle (oracle/lbm_oracle.c) to the reference itself (oracle/_ref, the
unmodified /root/reference sources) and to the committed golden fixtures, bitwise.
CPU only; sizes chosen so the whole file runs in seconds."""
import json
import os

import numpy as np
import pytest

from conftest import W, equal_bits, interior, random_pdf
from oracle.pyoracle import fnv1a64, make_snapshots, new_scratch

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALL_P = (1, 1, 1)


def test_equilibrium_frozen_values(oracle):
    """test_lattice_lbm.cpp:67-78."""
    feq = oracle.equilibrium(1.0, (0.05, 0.0, 0.0))
    assert abs(feq[0] - 0.99625 / 3.0) <= 1e-15 * feq[0]
    assert abs(feq[1] - 1.1575 / 18.0) <= 1e-15 * feq[1]
    assert abs(feq[2] - 0.8575 / 18.0) <= 1e-15 * feq[2]
    assert abs(feq[7] - 1.1575 / 36.0) <= 1e-15 * feq[7]
    assert abs(feq[15] - 0.99625 / 36.0) <= 1e-15 * feq[15]
    assert np.allclose(oracle.equilibrium(1.0, (0, 0, 0)), W, rtol=1e-15, atol=0)


def test_equilibrium_matches_reference(oracle, ref):
    rng = np.random.default_rng(0)
    for _ in range(50):
        rho = 0.9 + 0.2 * rng.random()
        u = 0.1 * (rng.random(3) - 0.5)
        assert equal_bits(oracle.equilibrium(rho, u), ref.equilibrium(rho, u))


@pytest.mark.parametrize("dims,fext", [((8, 8, 8), (1e-5, 0.0, -2e-5)), ((9, 5, 7), (0.0, 0.0, 0.0))])
def test_fused_sweep_matches_reference(oracle, ref, dims, fext):
    src = random_pdf(dims, seed=29)
    blk = ref.block(dims)
    blk.set_src(src)
    blk.fill_periodic(ALL_P)
    blk.sweep(0.8, fext, (0, 0, 0), dims)
    s = src.copy()
    d = np.zeros_like(s)
    oracle.fill_periodic(dims, s, ALL_P)
    assert equal_bits(s, blk.get_src())
    assert oracle.collide_stream(dims, s, d, 0.8, fext, (0, 0, 0), dims) == 0
    assert equal_bits(interior(d), interior(blk.get_dst()))


def test_stability_guard_counts(oracle, ref):
    dims = (4, 4, 4)
    s = np.zeros((19, 6, 6, 6))
    s[:, 1:-1, 1:-1, 1:-1] = W[:, None, None, None]
    s[1, 3, 3, 3] = 5.0
    oracle.fill_periodic(dims, s, ALL_P)
    bad = oracle.collide_stream(dims, s, np.zeros_like(s), 0.51, (0, 0, 0), (0, 0, 0), dims)
    assert bad > 0
    blk = ref.block(dims)
    blk.set_src(s)
    with pytest.raises(RuntimeError, match=f"fluid instability: {bad} cells"):
        blk.sweep(0.51, (0, 0, 0), (0, 0, 0), dims)


@pytest.mark.parametrize("case", range(3))
def test_boundaries_match_reference(oracle, ref, case):
    dims = (7, 6, 8)
    src = random_pdf(dims, seed=41 + case)
    kinds = [[1, 1, 1, 1, 2, 3], [0, 0, 1, 2, 0, 0], [1, 1, 3, 3, 2, 1]][case]
    touches = [[1] * 6, [1] * 6, [1, 0, 0, 1, 1, 0]][case]
    periodic = [tuple(int(kinds[2 * a] == 0) for a in range(3))][0]
    uw = np.zeros(18)
    uw[12:15] = (0.001, -0.002, 0.003)
    uw[6:9] = (0.01, 0.0, 0.002)
    rho = [1.0, 1.0, 1.02, 0.99, 1.0, 1.01]
    s = src.copy()
    oracle.fill_periodic(dims, s, periodic)
    oracle.apply_boundaries(dims, s, kinds, uw, rho, touches)
    blk = ref.block(dims)
    blk.set_src(src)
    blk.fill_periodic(periodic)
    blk.apply_boundaries(kinds, uw, rho, touches)
    assert equal_bits(s, blk.get_src())


def bed_snapshots(oracle, lo):
    rng = np.random.default_rng(7)
    centers = [(lo[0] + 10.3, lo[1] + 12.6, lo[2] + 11.2), (lo[0] + 19.0, lo[1] + 12.1, lo[2] + 12.0),
               (lo[0] + 28.4, lo[1] + 25.5, lo[2] + 30.1), (lo[0] - 3.0, lo[1] + 2.0, lo[2] + 2.0)]
    radii = [6.0, 5.0, 8.5, 5.5]
    return make_snapshots([2, 5, 9, 40], centers, radii, [oracle.f_of_r(r) for r in radii],
                          0.01 * (rng.random((4, 3)) - 0.5), 0.002 * (rng.random((4, 3)) - 0.5))


@pytest.mark.parametrize("lo", [(0, 0, 0), (16, 8, 24)])
def test_mapping_setu_psm_finalize_match_reference(oracle, ref, lo):
    dims = (36, 32, 40)
    s = bed_snapshots(oracle, lo)
    f_o, over = oracle.build_fraction_field(lo, dims, s)
    sv_o, unk = oracle.set_solid_velocities(lo, dims, s, f_o)
    assert over == 0 and unk == 0
    blk = ref.block(dims, lo)
    blk.set_snapshots(s)
    blk.map()
    blk.set_u()
    f_r = blk.get_fraction()
    c = f_r["count"]
    assert np.array_equal(c, f_o["count"]) and (c == 2).any()
    assert equal_bits(f_r["btot"], f_o["btot"])
    for e, (ik, bk) in enumerate((("id0", "b0"), ("id1", "b1"))):
        assert np.array_equal(f_r[ik][c > e], f_o[ik][c > e])
        assert equal_bits(f_r[bk][c > e], f_o[bk][c > e])
    sv_r = blk.get_svel()
    assert equal_bits(sv_r["v0"][c > 0], sv_o["v0"][c > 0])
    assert equal_bits(sv_r["v1"][c > 1], sv_o["v1"][c > 1])

    src = random_pdf(dims, seed=5)
    blk.set_src(src)
    blk.fill_periodic(ALL_P)
    blk.sweep(0.7, (0.0, 0.0, -1e-5), (0, 0, 0), dims, coupling=True)
    sc = src.copy()
    oracle.fill_periodic(dims, sc, ALL_P)
    d = np.zeros_like(sc)
    scr = new_scratch(dims)
    oracle.psm_collide_stream(dims, sc, d, 0.7, (0.0, 0.0, -1e-5), (0, 0, 0), dims, f_o, sv_o, scr)
    assert equal_bits(interior(d), interior(blk.get_dst()))
    scr_r = blk.get_scratch()
    assert equal_bits(scr_r["m0"][c > 0], scr["m0"][c > 0])
    ids_r, rows_r = blk.finalize(len(s["id"]))
    ids_o, rows_o = oracle.finalize_hydro(lo, dims, s, f_o, scr)
    assert list(ids_r) == list(ids_o)
    assert equal_bits(rows_r, rows_o)


def test_halo_self_messages_equal_periodic_fill(oracle):
    """sim.cpp:156-201 on a fully periodic single block: the 26 self-addressed slabs
    (source_slab(o) -> ghost_region(-o)) reproduce fill_periodic_ghosts exactly."""
    dims = (5, 4, 3)
    src = random_pdf(dims, seed=9, ghosts=False)
    halo = src.copy()
    for ox in (-1, 0, 1):
        for oy in (-1, 0, 1):
            for oz in (-1, 0, 1):
                off = (ox, oy, oz)
                if off == (0, 0, 0):
                    continue
                v = oracle.halo_pack(dims, src, off)
                assert v.size == 19 * np.prod([1 if o else d for o, d in zip(off, dims)])
                oracle.halo_unpack(dims, halo, tuple(-o for o in off), v)
    wrap = src.copy()
    oracle.fill_periodic(dims, wrap, ALL_P)
    assert equal_bits(halo, wrap)


def test_golden_fixtures(oracle):
    """tests/golden/golden.json: outputs of the reference itself (make_golden.py); arrays as
    FNV-1a hashes of their bytes, inputs regenerated from the recorded seeds."""
    g = json.load(open(os.path.join(GOLDEN, "golden.json")))
    h = lambda a: hex(fnv1a64(np.ascontiguousarray(a)))  # noqa: E731
    # fused forced sweep, 8^3 random periodic field
    dims = tuple(g["sweep_dims"])
    s = random_pdf(dims, seed=g["seeds"]["sweep_src"])
    d = np.zeros_like(s)
    oracle.fill_periodic(dims, s, ALL_P)
    oracle.collide_stream(dims, s, d, g["sweep_tau"], g["sweep_fext"], (0, 0, 0), dims)
    assert h(interior(d)) == g["sweep_out_fnv"]
    # bed boundary fill (no-slip sides, velocity inflow, pressure outflow)
    dims = tuple(g["bc_dims"])
    s = random_pdf(dims, seed=g["seeds"]["bc_src"])
    oracle.apply_boundaries(dims, s, g["bc_kinds"], g["bc_uwall"], g["bc_rho"], [1] * 6)
    assert h(s) == g["bc_out_fnv"]
    # two overlapping moving spheres: mapping, setU, PSM step, partials
    snaps = make_snapshots(g["map_ids"], g["map_x"], g["map_r"], g["map_fr"], g["map_u"], g["map_w"])
    dims = tuple(g["map_dims"])
    f, _ = oracle.build_fraction_field((0, 0, 0), dims, snaps)
    assert h(f["count"]) == g["map_count_fnv"] and h(f["btot"]) == g["map_btot_fnv"]
    sv, _ = oracle.set_solid_velocities((0, 0, 0), dims, snaps, f)
    s = random_pdf(dims, seed=g["seeds"]["map_src"])
    oracle.fill_periodic(dims, s, ALL_P)
    d = np.zeros_like(s)
    scr = new_scratch(dims)
    oracle.psm_collide_stream(dims, s, d, g["map_tau"], (0, 0, 0), (0, 0, 0), dims, f, sv, scr)
    assert h(interior(d)) == g["map_out_fnv"]
    ids, rows = oracle.finalize_hydro((0, 0, 0), dims, snaps, f, scr)
    assert list(ids) == g["map_partial_ids"]
    assert equal_bits(rows, np.array(g["map_partials"]))


def test_survey_known_answers_config1(ref):
    """SURVEY.md §8(c) known answers of the reference on config 1 (64^3 settling sphere)."""
    ka = json.load(open(os.path.join(GOLDEN, "config1_known_answers.json")))
    sim = ref.sim(ka["config"])
    sim.run(10)
    assert hex(fnv1a64(sim.pdfs())) == ka["steps"]["10"]["pdf_hash"]
    p = sim.particles()[0]
    assert p[3] == ka["steps"]["10"]["x_z"]
    assert p[6] == ka["steps"]["10"]["u_z"]
    assert p[12] == ka["steps"]["10"]["f_hydro_z"]


def _neumaier(values):
    """CompensatedSum (vec3.hpp:71-95) in iteration order: Neumaier add, value = sum + comp."""
    s = c = 0.0
    for v in values:
        t = s + v
        c += (s - t) + v if abs(s) >= abs(v) else (v - t) + s
        s = t
    return s + c


def test_moments_restatement_pinned_to_total_mass_momentum(oracle):
    """Oracle.moments (per-cell rho and bare momentum, the sums of lbm.cpp:61-93) summed in the
    reference's serial order reproduces total_mass / total_momentum of the C restatement
    bitwise, which test_fused_sweep_matches_reference pins to the reference."""
    dims = (7, 5, 6)
    src = random_pdf(dims, seed=12)
    mom = oracle.moments(dims, src).reshape(-1, 4)
    assert equal_bits(np.float64(_neumaier(mom[:, 0])), np.float64(oracle.total_mass(dims, src)))
    tm = oracle.total_momentum(dims, src)
    for a in range(3):
        assert equal_bits(np.float64(_neumaier(mom[:, 1 + a])), np.float64(tm[a]))


def test_reference_observers_shim(ref):
    """oracle/_ref exposes io::sample_scalars / write_grid_dump (the drop-in observer checks):
    the sampled mass is the simulation's total_fluid_mass, the dump has one line per cell."""
    import tempfile
    ka = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "config1_known_answers.json")))
    cfg = json.loads(ka["config"])
    cfg["domain"] = [16, 16, 16]
    cfg["particles"] = {"count": 0}
    sim = ref.sim(json.dumps(cfg))
    sim.run(1)
    obs = sim.observe()
    assert obs[0] == 1 and equal_bits(np.float64(obs[1]), np.float64(sim.mass()))
    with tempfile.TemporaryDirectory() as d:
        sim.grid_dump(os.path.join(d, "g.dat"))
        lines = open(os.path.join(d, "g.dat")).read().splitlines()
    assert lines[1] == "# columns: x y z rho ux uy uz B" and len(lines) == 2 + 16 ** 3
