"""TEST INFRASTRUCTURE — numpy/ctypes front ends of the two parity checkers.

Arrays use the reference layouts (see ``lbm_oracle.h``):

* PDF buffers: ``float64[19, nz+2, ny+2, nx+2]`` (C order == ``PdfField::idx``, field.hpp:47-49)
* fraction / velocity / scratch: interior lexicographic ``[nz, ny, nx]`` (+ trailing 3 for Vec3)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblbdem_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i3 = C.c_int * 3
_d3 = C.c_double * 3

# D3Q19 velocity set in the reference's order (lattice.hpp:18-29: rest, then opposite pairs)
LATTICE_C = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1),
             (1, 1, 0), (-1, -1, 0), (1, -1, 0), (-1, 1, 0), (1, 0, 1), (-1, 0, -1),
             (1, 0, -1), (-1, 0, 1), (0, 1, 1), (0, -1, -1), (0, 1, -1), (0, -1, 1)]

# status codes shared with include/lbg.h and oracle/ref_shim.cpp
CONFIG_ERROR, NUMERIC_ERROR, SYNC_ERROR, IO_ERROR = 1, 2, 3, 4


def build_oracle() -> None:
    """Compile liboracle.so (gcc; part of __graft_entry__.build())."""
    subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])


def build_ref() -> bool:
    """Compile oracle/_ref from /root/reference sources when they are present."""
    if not os.path.isdir("/root/reference/proj/src"):
        return os.path.exists(REF_SO)
    subprocess.check_call(["make", "-s", "-j8", "-C", HERE, "ref"])
    return True


def pdf_shape(dims):
    nx, ny, nz = dims
    return (19, nz + 2, ny + 2, nx + 2)


def new_pdf(dims):
    return np.zeros(pdf_shape(dims), dtype=np.float64)


class Oracle:
    """Plain-C restatement (oracle/lbm_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build_oracle()
        L = self.L = C.CDLL(path)
        L.orc_collide_stream.restype = C.c_long
        L.orc_collide_stream.argtypes = [C.c_int] * 3 + [_dp, _dp, C.c_double, _d3, _i3, _i3]
        L.orc_stream.argtypes = [C.c_int] * 3 + [_dp, _dp, _i3, _i3]
        L.orc_psm_collide_stream.restype = C.c_long
        L.orc_psm_collide_stream.argtypes = [C.c_int] * 3 + [
            _dp, _dp, C.c_double, _d3, _i3, _i3, _u8, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc_fill_periodic.argtypes = [C.c_int] * 3 + [_dp, _i3]
        L.orc_apply_boundaries.argtypes = [C.c_int] * 3 + [
            _dp, C.c_int * 6, C.c_double * 18, C.c_double * 6, C.c_int * 6]
        L.orc_equilibrium.argtypes = [C.c_double, _d3, _dp]
        L.orc_f_of_r.restype = C.c_double
        L.orc_f_of_r.argtypes = [C.c_double]
        L.orc_sphere_volume.restype = C.c_double
        L.orc_sphere_volume.argtypes = [C.c_double]
        L.orc_build_fraction_field.restype = C.c_long
        L.orc_build_fraction_field.argtypes = [_i3, _i3, C.c_int, _ip, _dp, _dp, _dp, C.c_int,
                                               _u8, _ip, _ip, _dp, _dp, _dp]
        L.orc_set_solid_velocities.restype = C.c_long
        L.orc_set_solid_velocities.argtypes = [_i3, _i3, C.c_int, _ip, _dp, _dp, _dp,
                                               _u8, _ip, _ip, _dp, _dp]
        L.orc_finalize_hydro.restype = C.c_int
        L.orc_finalize_hydro.argtypes = [_i3, _i3, C.c_int, _ip, _dp, _u8, _ip, _ip, _dp, _dp,
                                         _ip, _dp]
        L.orc_halo_pack.restype = C.c_long
        L.orc_halo_pack.argtypes = [C.c_int] * 3 + [_dp, _i3, _dp]
        L.orc_halo_unpack.restype = C.c_long
        L.orc_halo_unpack.argtypes = [C.c_int] * 3 + [_dp, _i3, _dp]
        L.orc_total_mass.restype = C.c_double
        L.orc_total_mass.argtypes = [C.c_int] * 3 + [_dp]
        L.orc_total_momentum.argtypes = [C.c_int] * 3 + [_dp, _dp]

    # -- fluid ---------------------------------------------------------------
    def equilibrium(self, rho, u):
        out = np.zeros(19)
        self.L.orc_equilibrium(rho, _d3(*u), out)
        return out

    def collide_stream(self, dims, src, dst, tau, fext, lo, hi):
        return self.L.orc_collide_stream(*dims, src, dst, tau, _d3(*fext), _i3(*lo), _i3(*hi))

    def stream(self, dims, src, dst, lo, hi):
        self.L.orc_stream(*dims, src, dst, _i3(*lo), _i3(*hi))

    def psm_collide_stream(self, dims, src, dst, tau, fext, lo, hi, frac, svel, scratch):
        return self.L.orc_psm_collide_stream(
            *dims, src, dst, tau, _d3(*fext), _i3(*lo), _i3(*hi), frac["count"], frac["b0"],
            frac["b1"], frac["btot"], svel["v0"], svel["v1"], scratch["m0"], scratch["m1"])

    def fill_periodic(self, dims, src, periodic):
        self.L.orc_fill_periodic(*dims, src, _i3(*[int(bool(p)) for p in periodic]))

    def apply_boundaries(self, dims, src, kinds, uwall, rho, touches):
        self.L.orc_apply_boundaries(*dims, src, (C.c_int * 6)(*kinds),
                                    (C.c_double * 18)(*np.ravel(uwall)), (C.c_double * 6)(*rho),
                                    (C.c_int * 6)(*[int(bool(t)) for t in touches]))

    def total_mass(self, dims, src):
        return self.L.orc_total_mass(*dims, src)

    def total_momentum(self, dims, src):
        out = np.zeros(3)
        self.L.orc_total_momentum(*dims, src, out)
        return out

    @staticmethod
    def moments(dims, src):
        """Per-cell {rho, mx, my, mz}, shape (nz, ny, nx, 4), in the reference's sum order:
        rho = 0 + f_0 + ... + f_18, m = 0 + f_q * c_q for q = 0..18 (lbm.hpp:55-60,
        lbm.cpp:61-67 / 82-91). Elementwise numpy, so each cell's arithmetic is exactly that."""
        nx, ny, nz = dims
        f = src[:, 1:nz + 1, 1:ny + 1, 1:nx + 1]
        out = np.zeros((nz, ny, nx, 4))
        rho = np.zeros((nz, ny, nx))
        m = [np.zeros((nz, ny, nx)) for _ in range(3)]
        for q in range(19):
            rho = rho + f[q]
            for a in range(3):
                m[a] = m[a] + f[q] * float(LATTICE_C[q][a])
        out[..., 0] = rho
        for a in range(3):
            out[..., 1 + a] = m[a]
        return out

    # -- coupling ------------------------------------------------------------
    def f_of_r(self, r):
        return self.L.orc_f_of_r(r)

    def sphere_volume(self, r):
        return self.L.orc_sphere_volume(r)

    def build_fraction_field(self, lo, dims, snaps, subdivisions=8, frac=None):
        if frac is None:
            frac = new_fraction(dims)
        over = self.L.orc_build_fraction_field(
            _i3(*lo), _i3(*dims), len(snaps["id"]), snaps["id"], snaps["x"], snaps["r"],
            snaps["f_r"], subdivisions, frac["count"], frac["id0"], frac["id1"], frac["b0"],
            frac["b1"], frac["btot"])
        return frac, over

    def set_solid_velocities(self, lo, dims, snaps, frac, svel=None):
        if svel is None:
            svel = new_svel(dims)
        unk = self.L.orc_set_solid_velocities(
            _i3(*lo), _i3(*dims), len(snaps["id"]), snaps["id"], snaps["x"], snaps["u"],
            snaps["w"], frac["count"], frac["id0"], frac["id1"], svel["v0"], svel["v1"])
        return svel, unk

    def finalize_hydro(self, lo, dims, snaps, frac, scratch):
        n = len(snaps["id"])
        used = np.zeros(max(n, 1), dtype=np.int32)
        rows = np.zeros((max(n, 1), 12))
        rc = self.L.orc_finalize_hydro(_i3(*lo), _i3(*dims), n, snaps["id"], snaps["x"],
                                       frac["count"], frac["id0"], frac["id1"], scratch["m0"],
                                       scratch["m1"], used, rows)
        if rc != 0:
            raise SyncErrorOracle("hydrodynamic force for unknown particle id")
        sel = np.nonzero(used[:n])[0]
        return snaps["id"][sel].copy(), rows[sel].copy()

    def halo_pack(self, dims, src, off):
        n = 19 * _slab_cells(dims, off)
        out = np.zeros(n)
        self.L.orc_halo_pack(*dims, src, _i3(*off), out)
        return out

    def halo_unpack(self, dims, src, direction, values):
        self.L.orc_halo_unpack(*dims, src, _i3(*direction), np.ascontiguousarray(values))


class SyncErrorOracle(RuntimeError):
    pass


def _slab_cells(dims, off):
    n = 1
    for a in range(3):
        n *= 1 if off[a] != 0 else dims[a]
    return n


def new_fraction(dims):
    nx, ny, nz = dims
    shp = (nz, ny, nx)
    return {"count": np.zeros(shp, np.uint8), "id0": np.full(shp, -1, np.int32),
            "id1": np.full(shp, -1, np.int32), "b0": np.zeros(shp), "b1": np.zeros(shp),
            "btot": np.zeros(shp)}


def new_svel(dims):
    nx, ny, nz = dims
    return {"v0": np.zeros((nz, ny, nx, 3)), "v1": np.zeros((nz, ny, nx, 3))}


def new_scratch(dims):
    nx, ny, nz = dims
    return {"m0": np.zeros((nz, ny, nx, 3)), "m1": np.zeros((nz, ny, nx, 3))}


def make_snapshots(ids, x, r, f_r, u=None, w=None):
    n = len(ids)
    return {"id": np.ascontiguousarray(ids, dtype=np.int32),
            "x": np.ascontiguousarray(np.reshape(x, (n, 3)), dtype=np.float64),
            "r": np.ascontiguousarray(r, dtype=np.float64),
            "f_r": np.ascontiguousarray(f_r, dtype=np.float64),
            "u": np.ascontiguousarray(np.zeros((n, 3)) if u is None else np.reshape(u, (n, 3)), dtype=np.float64),
            "w": np.ascontiguousarray(np.zeros((n, 3)) if w is None else np.reshape(w, (n, 3)), dtype=np.float64)}


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class RefLib:
    """The unmodified reference (oracle/_ref/liblbdem_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
        L = self.L = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_block_create.restype = vp
        L.ref_block_create.argtypes = [_i3, _i3]
        L.ref_block_destroy.argtypes = [vp]
        L.ref_alloc_cells.restype = C.c_long
        L.ref_alloc_cells.argtypes = [vp]
        for n in ("ref_get_src", "ref_set_src", "ref_get_dst", "ref_set_dst"):
            getattr(L, n).argtypes = [vp, _dp]
        L.ref_swap.argtypes = [vp]
        L.ref_fill_periodic.argtypes = [vp, _i3]
        L.ref_apply_boundaries.argtypes = [vp, C.c_int * 6, C.c_double * 18, C.c_double * 6,
                                           C.c_int * 6]
        L.ref_sweep.argtypes = [vp, C.c_double, _d3, _i3, _i3, C.c_int, C.c_int]
        L.ref_stream.argtypes = [vp, _i3, _i3]
        L.ref_equilibrium.argtypes = [C.c_double, _d3, _dp]
        L.ref_total_mass.argtypes = [vp, C.POINTER(C.c_double)]
        L.ref_total_momentum.argtypes = [vp, _dp]
        L.ref_f_of_r.argtypes = [C.c_double, C.POINTER(C.c_double)]
        L.ref_sphere_volume.restype = C.c_double
        L.ref_sphere_volume.argtypes = [C.c_double]
        L.ref_set_snapshots.argtypes = [vp, C.c_int, _ip, _dp, _dp, _dp, _dp, _dp]
        L.ref_map.argtypes = [vp, C.c_int, C.c_int]
        L.ref_set_u.argtypes = [vp, C.c_int]
        L.ref_frac_cells.restype = C.c_long
        L.ref_frac_cells.argtypes = [vp]
        L.ref_get_fraction.argtypes = [vp, _u8, _ip, _ip, _dp, _dp, _dp]
        L.ref_set_fraction.argtypes = [vp, _u8, _ip, _ip, _dp, _dp, _dp]
        for n in ("ref_get_svel", "ref_set_svel", "ref_get_scratch", "ref_set_scratch"):
            getattr(L, n).argtypes = [vp, _dp, _dp]
        L.ref_finalize.argtypes = [vp, C.POINTER(C.c_int), _ip, _dp]
        L.ref_sim_create.restype = vp
        L.ref_sim_create.argtypes = [C.c_char_p]
        L.ref_sim_destroy.argtypes = [vp]
        L.ref_sim_run.argtypes = [vp, C.c_long]
        L.ref_sim_add_particles.argtypes = [vp, C.c_int, _dp]
        L.ref_sim_params.argtypes = [vp, C.POINTER(C.c_double), _dp, _ip]
        L.ref_sim_shear_wave.argtypes = [vp]
        L.ref_sim_pdfs.argtypes = [vp, _dp]
        L.ref_sim_num_particles.restype = C.c_int
        L.ref_sim_num_particles.argtypes = [vp]
        L.ref_sim_particles.argtypes = [vp, _dp]
        L.ref_sim_mass.restype = C.c_double
        L.ref_sim_mass.argtypes = [vp]
        L.ref_sim_observe.argtypes = [vp, _dp]
        L.ref_sim_grid_dump.argtypes = [vp, C.c_char_p]
        L.ref_sim_reset_timers.argtypes = [vp]
        L.ref_sim_timings.argtypes = [vp, _dp]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_max_threads.restype = C.c_int

    def check(self, rc):
        if rc != 0:
            raise RefError(rc, self.L.ref_last_error().decode())

    def set_threads(self, n):
        self.L.ref_set_threads(int(n))

    def equilibrium(self, rho, u):
        out = np.zeros(19)
        self.L.ref_equilibrium(rho, _d3(*u), out)
        return out

    def f_of_r(self, r):
        v = C.c_double()
        self.check(self.L.ref_f_of_r(r, C.byref(v)))
        return v.value

    def block(self, dims, lo=(0, 0, 0)):
        return RefBlock(self, lo, dims)

    def sim(self, cfg_json: str):
        h = self.L.ref_sim_create(cfg_json.encode())
        if not h:
            raise RefError(-1, self.L.ref_last_error().decode())
        return RefSim(self, h)


class RefBlock:
    def __init__(self, lib: RefLib, lo, dims):
        self.lib, self.L = lib, lib.L
        self.lo, self.dims = tuple(lo), tuple(dims)
        self.h = self.L.ref_block_create(_i3(*lo), _i3(*dims))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.ref_block_destroy(self.h)
            self.h = None

    def get_src(self):
        a = new_pdf(self.dims)
        self.L.ref_get_src(self.h, a)
        return a

    def set_src(self, a):
        self.L.ref_set_src(self.h, np.ascontiguousarray(a, dtype=np.float64))

    def get_dst(self):
        a = new_pdf(self.dims)
        self.L.ref_get_dst(self.h, a)
        return a

    def set_dst(self, a):
        self.L.ref_set_dst(self.h, np.ascontiguousarray(a, dtype=np.float64))

    def swap(self):
        self.L.ref_swap(self.h)

    def fill_periodic(self, periodic):
        self.lib.check(self.L.ref_fill_periodic(self.h, _i3(*[int(bool(p)) for p in periodic])))

    def apply_boundaries(self, kinds, uwall, rho, touches):
        self.lib.check(self.L.ref_apply_boundaries(
            self.h, (C.c_int * 6)(*kinds), (C.c_double * 18)(*np.ravel(uwall)),
            (C.c_double * 6)(*rho), (C.c_int * 6)(*[int(bool(t)) for t in touches])))

    def sweep(self, tau, fext, lo, hi, coupling=False, omp=False):
        self.lib.check(self.L.ref_sweep(self.h, tau, _d3(*fext), _i3(*lo), _i3(*hi),
                                        int(coupling), int(omp)))

    def stream(self, lo, hi):
        self.lib.check(self.L.ref_stream(self.h, _i3(*lo), _i3(*hi)))

    def total_mass(self):
        v = C.c_double()
        self.lib.check(self.L.ref_total_mass(self.h, C.byref(v)))
        return v.value

    def set_snapshots(self, s):
        self.L.ref_set_snapshots(self.h, len(s["id"]), s["id"], s["x"], s["r"], s["f_r"],
                                 s["u"], s["w"])

    def map(self, subdivisions=8, omp=False):
        self.lib.check(self.L.ref_map(self.h, subdivisions, int(omp)))

    def set_u(self, omp=False):
        self.lib.check(self.L.ref_set_u(self.h, int(omp)))

    def get_fraction(self):
        f = new_fraction(self.dims)
        self.L.ref_get_fraction(self.h, f["count"], f["id0"], f["id1"], f["b0"], f["b1"], f["btot"])
        return f

    def set_fraction(self, f):
        self.L.ref_set_fraction(self.h, f["count"], f["id0"], f["id1"], f["b0"], f["b1"], f["btot"])

    def get_svel(self):
        s = new_svel(self.dims)
        self.L.ref_get_svel(self.h, s["v0"], s["v1"])
        return s

    def set_svel(self, s):
        self.L.ref_set_svel(self.h, np.ascontiguousarray(s["v0"]), np.ascontiguousarray(s["v1"]))

    def get_scratch(self):
        s = new_scratch(self.dims)
        self.L.ref_get_scratch(self.h, s["m0"], s["m1"])
        return s

    def set_scratch(self, s):
        self.L.ref_set_scratch(self.h, np.ascontiguousarray(s["m0"]), np.ascontiguousarray(s["m1"]))

    def finalize(self, n_snaps):
        n = C.c_int()
        ids = np.zeros(max(n_snaps, 1), np.int32)
        rows = np.zeros((max(n_snaps, 1), 12))
        self.lib.check(self.L.ref_finalize(self.h, C.byref(n), ids, rows))
        return ids[: n.value].copy(), rows[: n.value].copy()


class RefSim:
    def __init__(self, lib: RefLib, h):
        self.lib, self.L, self.h = lib, lib.L, h
        tau = C.c_double()
        fext = np.zeros(3)
        dom = np.zeros(3, np.int32)
        self.L.ref_sim_params(h, C.byref(tau), fext, dom)
        self.tau, self.fext, self.domain = tau.value, fext, tuple(int(d) for d in dom)

    def close(self):
        if getattr(self, "h", None):
            self.L.ref_sim_destroy(self.h)
            self.h = None

    __del__ = close

    def run(self, steps):
        self.lib.check(self.L.ref_sim_run(self.h, steps))

    def add_particles(self, rows):
        """rows: (n, 6) of id, x, y, z, r, m (Simulation::add_particles)"""
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        self.lib.check(self.L.ref_sim_add_particles(self.h, len(rows), rows))

    def shear_wave(self):
        self.L.ref_sim_shear_wave(self.h)

    def pdfs(self):
        nx, ny, nz = self.domain
        a = np.zeros((nz, ny, nx, 19))
        self.L.ref_sim_pdfs(self.h, a)
        return a

    def particles(self):
        n = self.L.ref_sim_num_particles(self.h)
        rows = np.zeros((max(n, 1), 16))
        if n:
            self.L.ref_sim_particles(self.h, rows)
        return rows[:n]

    def mass(self):
        return self.L.ref_sim_mass(self.h)

    def observe(self):
        """io::sample_scalars: [step, mass, px, py, pz, fluid_ke, particle_ke, min_gap, max_u]."""
        out = np.zeros(9)
        self.lib.check(self.L.ref_sim_observe(self.h, out))
        return out

    def grid_dump(self, path):
        self.lib.check(self.L.ref_sim_grid_dump(self.h, str(path).encode()))

    def reset_timers(self):
        self.L.ref_sim_reset_timers(self.h)

    def timings(self):
        out = np.zeros(8)
        self.L.ref_sim_timings(self.h, out)
        return out


def fnv1a64(arr) -> int:
    """FNV-1a 64 over the raw bytes of ``arr`` (hash SURVEY §8(c) quotes for config 1)."""
    a = np.ascontiguousarray(arr).view(np.uint8).ravel()
    L = Oracle().L
    L.orc_fnv1a64.restype = C.c_uint64
    L.orc_fnv1a64.argtypes = [_u8, C.c_long]
    return int(L.orc_fnv1a64(a, a.size))
