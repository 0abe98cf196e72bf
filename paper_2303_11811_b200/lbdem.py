"""Host-side mirror of the reference operator API (namespace ``lbdem``), backed by liblbg.

Names, argument meaning and error behaviour follow the reference C++ library so a caller
of ``lbm::collide_stream_omp`` / ``psm::build_fraction_field`` / ``lbm::apply_boundaries``
finds the same operation here (citations are to /root/reference/proj):

====================================  =============================================
reference                              here
====================================  =============================================
errors.hpp ConfigError/NumericError/…  ConfigError / NumericError / SyncError / IoError
field.hpp CellBox, boundary_shell      CellBox, boundary_shell
lbm.hpp FluidParams                    FluidParams
boundary.hpp BcKind/FaceBc/BcSpec      BcKind / FaceBc / BcSpec
psm.hpp ParticleSnapshot/HydroPartial  ParticleSnapshot / HydroPartial
BlockState fields (sim.hpp:28-52)      Block (device PdfField + coupling fields)
lbm::collide_stream_{serial,omp}       collide_stream(block, params, box)
psm::psm_collide_stream_{serial,omp}   psm_collide_stream(block, params, box)
lbm::fill_periodic_ghosts              fill_periodic_ghosts(block, periodic)
lbm::apply_boundaries                  apply_boundaries(block, spec, touches)
psm::build_fraction_field (+registry)  build_fraction_field(block, snapshots)
psm::set_solid_velocities              set_solid_velocities(block, snapshots)
psm::finalize_hydro_forces             finalize_hydro_forces(block)
psm::f_of_r                            f_of_r(r)   (host, like the reference)
lbm::total_mass / total_momentum       Block.total_mass / total_momentum
lbm::cell_macroscopic (observers)      Block.moments (per-cell rho, bare momentum, B)
io::sample_scalars (fluid part)        Block.observe (one device reduction)
begin/complete_halo_exchange           Block.halo_stage / halo_fetch (device to device)
====================================  =============================================

Like the reference operators, the free functions complete the operation and raise at the
end (they call ``Block.sync()``); the ``Block`` methods are the asynchronous C-ABI calls a
step driver batches between phase barriers.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Sequence

import numpy as np

from . import lbg as _abi

Q = 19


# --------------------------------------------------------------------------- errors
class ConfigError(RuntimeError):
    """errors.hpp:10-14 (CLI exit code 2)."""


class NumericError(RuntimeError):
    """errors.hpp:16-20 (CLI exit code 3)."""


class SyncError(RuntimeError):
    """errors.hpp:22-27 (CLI exit code 3)."""


class IoError(RuntimeError):
    """errors.hpp:29-32 (CLI exit code 4)."""


class CudaError(RuntimeError):
    """CUDA / NCCL failure inside liblbg (no reference twin)."""


_EXC = {_abi.CONFIG_ERROR: ConfigError, _abi.NUMERIC_ERROR: NumericError,
        _abi.SYNC_ERROR: SyncError, _abi.IO_ERROR: IoError, _abi.CUDA_ERROR: CudaError,
        _abi.INVALID: ValueError}


def _lib():
    return _abi.load()


def check(status: int) -> None:
    if status != _abi.OK:
        msg = _lib().lbg_last_error().decode()
        raise _EXC.get(status, RuntimeError)(msg)


# --------------------------------------------------------------------------- value types
@dataclass(frozen=True)
class CellBox:
    """field.hpp:13-30 — half-open box [lo, hi)."""
    lo: tuple
    hi: tuple

    def empty(self) -> bool:
        return any(h <= l for l, h in zip(self.lo, self.hi))

    def volume(self) -> int:
        return 0 if self.empty() else int(np.prod([h - l for l, h in zip(self.lo, self.hi)]))

    def c(self) -> _abi.Box:
        return _abi.Box((C.c_int * 3)(*self.lo), (C.c_int * 3)(*self.hi))


def boundary_shell(dims: Sequence[int], width: int = 1) -> list[CellBox]:
    """field.cpp:55-72 — z slabs, then y slabs, then x slabs."""
    dx, dy, dz = dims
    w = width
    if dx <= 2 * w or dy <= 2 * w or dz <= 2 * w:
        return [CellBox((0, 0, 0), tuple(dims))]
    return [CellBox((0, 0, 0), (dx, dy, w)), CellBox((0, 0, dz - w), (dx, dy, dz)),
            CellBox((0, 0, w), (dx, w, dz - w)), CellBox((0, dy - w, w), (dx, dy, dz - w)),
            CellBox((0, w, w), (w, dy - w, dz - w)), CellBox((dx - w, w, w), (dx, dy - w, dz - w))]


@dataclass
class FluidParams:
    """lbm.hpp:21-33."""
    tau: float = 1.0
    f_ext: tuple = (0.0, 0.0, 0.0)

    def nu(self) -> float:
        return (self.tau - 0.5) / 3.0

    def omega(self) -> float:
        return 1.0 / self.tau

    def validate(self) -> None:
        if not self.tau > 0.5:
            raise ConfigError(f"fluid relaxation time tau must be > 0.5 (got {self.tau:f})")

    def c(self) -> _abi.Fluid:
        return _abi.Fluid(self.tau, (C.c_double * 3)(*self.f_ext))


class BcKind(IntEnum):
    """boundary.hpp:11."""
    periodic = _abi.BC_PERIODIC
    no_slip = _abi.BC_NO_SLIP
    velocity = _abi.BC_VELOCITY
    pressure = _abi.BC_PRESSURE


@dataclass
class FaceBc:
    """boundary.hpp:13-17."""
    kind: BcKind = BcKind.periodic
    u_wall: tuple = (0.0, 0.0, 0.0)
    rho: float = 1.0


@dataclass
class BcSpec:
    """boundary.hpp:22-31; faces in order -x,+x,-y,+y,-z,+z."""
    faces: list = field(default_factory=lambda: [FaceBc() for _ in range(6)])

    def periodic_axis(self, axis: int) -> bool:
        return (self.faces[2 * axis].kind == BcKind.periodic and
                self.faces[2 * axis + 1].kind == BcKind.periodic)

    def validate(self) -> None:
        for axis in range(3):
            lo = self.faces[2 * axis].kind == BcKind.periodic
            hi = self.faces[2 * axis + 1].kind == BcKind.periodic
            if lo != hi:
                raise ConfigError(f"periodic boundary must be assigned to both faces of axis {axis}")

    def c(self):
        arr = (_abi.FaceBc * 6)()
        for f, fb in enumerate(self.faces):
            arr[f].kind = int(fb.kind)
            arr[f].u_wall = (C.c_double * 3)(*fb.u_wall)
            arr[f].rho = fb.rho
        return arr


@dataclass
class ParticleSnapshot:
    """psm.hpp:16-23."""
    id: int
    x: tuple
    r: float
    f_r: float
    u: tuple = (0.0, 0.0, 0.0)
    omega: tuple = (0.0, 0.0, 0.0)


@dataclass
class HydroPartial:
    """psm.hpp:88-92."""
    id: int
    f: np.ndarray
    f_comp: np.ndarray
    t: np.ndarray
    t_comp: np.ndarray


def snapshot_array(snaps) -> "C.Array":
    """ParticleSnapshot list (or a dict of numpy columns) -> lbg_snapshot[]."""
    if isinstance(snaps, dict):
        n = len(snaps["id"])
        arr = (_abi.Snapshot * max(n, 1))()
        for i in range(n):
            s = arr[i]
            s.id = int(snaps["id"][i])
            s.x = (C.c_double * 3)(*snaps["x"][i])
            s.r = float(snaps["r"][i])
            s.f_r = float(snaps["f_r"][i])
            s.u = (C.c_double * 3)(*snaps["u"][i])
            s.omega = (C.c_double * 3)(*snaps["w"][i])
        return arr, n
    n = len(snaps)
    arr = (_abi.Snapshot * max(n, 1))()
    for i, sp in enumerate(snaps):
        arr[i].id = sp.id
        arr[i].x = (C.c_double * 3)(*sp.x)
        arr[i].r = sp.r
        arr[i].f_r = sp.f_r
        arr[i].u = (C.c_double * 3)(*sp.u)
        arr[i].omega = (C.c_double * 3)(*sp.omega)
    return arr, n


# --------------------------------------------------------------------------- psm host math
def sphere_over_unit_square_volume(r: float) -> float:
    """psm.cpp:12-18 (host-side, like the reference; uploaded as f_r)."""
    r2 = r * r
    s = math.sqrt(r2 - 0.5)
    return ((1.0 / 12.0 - r2) * math.atan(0.5 * s / (0.5 - r2)) + s / 3.0 +
            (r2 - 1.0 / 12.0) * math.atan(0.5 / s) - (4.0 / 3.0) * r2 * r * math.atan(0.25 / (r * s)))


def f_of_r(r: float) -> float:
    """psm.cpp:20-26."""
    if not r >= math.sqrt(0.5):
        raise ConfigError(f"particle radius {r:f} below mapping validity floor sqrt(1/2)")
    return sphere_over_unit_square_volume(r) - r + 0.5


# --------------------------------------------------------------------------- device block
def _ptr(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


class Block:
    """Device twin of a reference BlockState's fields (sim.hpp:28-52)."""

    def __init__(self, dims, lo=(0, 0, 0), coupling=False, device=0):
        self.dims = tuple(int(d) for d in dims)
        self.lo = tuple(int(v) for v in lo)
        self.coupling = bool(coupling)
        h = C.c_void_p()
        check(_lib().lbg_block_create(device, (C.c_int * 3)(*self.lo), (C.c_int * 3)(*self.dims),
                                      int(coupling), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            _lib().lbg_block_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # shapes
    @property
    def pdf_shape(self):
        nx, ny, nz = self.dims
        return (Q, nz + 2, ny + 2, nx + 2)

    @property
    def cells(self):
        nx, ny, nz = self.dims
        return nx * ny * nz

    @property
    def stream(self) -> int:
        return _lib().lbg_block_stream(self.h) or 0

    # PdfField access
    def upload_src(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        assert a.shape == self.pdf_shape
        check(_lib().lbg_upload_src(self.h, _ptr(a)))

    def download_src(self):
        a = np.empty(self.pdf_shape)
        check(_lib().lbg_download_src(self.h, _ptr(a)))
        return a

    def upload_dst(self, a):
        a = np.ascontiguousarray(a, dtype=np.float64)
        assert a.shape == self.pdf_shape
        check(_lib().lbg_upload_dst(self.h, _ptr(a)))

    def download_dst(self):
        a = np.empty(self.pdf_shape)
        check(_lib().lbg_download_dst(self.h, _ptr(a)))
        return a

    def fill_equilibrium(self, rho, u):
        check(_lib().lbg_fill_equilibrium(self.h, rho, (C.c_double * 3)(*u)))

    def init_shear_wave(self, domain):
        check(_lib().lbg_init_shear_wave(self.h, (C.c_int * 3)(*domain)))

    def fill_ghosts_src(self, v):
        check(_lib().lbg_fill_ghosts_src(self.h, v))

    def swap(self):
        check(_lib().lbg_swap(self.h))

    def run_host(self, params: FluidParams, host, steps: int, slab_planes: int = 0) -> dict:
        """Simulation::run(steps) (sim.cpp:702-704) of this fully periodic plain block on a
        host PdfField `host` (pdf_shape, float64, C order; pinned memory for overlapped
        copies), in place: upload, sweeps and download pipelined over z-slabs (lbg_run_host).
        Interior cells receive the state after `steps` steps; ghost cells are left as they
        were. Returns the accumulated error counters (NumericError raised like sync())."""
        assert host.shape == self.pdf_shape and host.dtype == np.float64 and host.flags.c_contiguous
        fl, e = params.c(), _abi.Errors()
        check(_lib().lbg_run_host(self.h, C.byref(fl), _ptr(host), int(steps), int(slab_planes), C.byref(e)))
        return {"unstable": e.unstable_cells, "overfull": e.overfull_cells, "unknown": e.unknown_ids}

    # operators (async)
    def sweep(self, params: FluidParams, box: CellBox):
        fl, bx = params.c(), box.c()
        check(_lib().lbg_sweep(self.h, C.byref(fl), C.byref(bx)))

    def sweep_boxes(self, params: FluidParams, boxes: Sequence[CellBox]):
        fl = params.c()
        arr = (_abi.Box * max(len(boxes), 1))(*[b.c() for b in boxes])
        check(_lib().lbg_sweep_boxes(self.h, C.byref(fl), arr, len(boxes)))

    def set_periodic_wrap(self, wrap):
        """Periodic axes the sweep wraps in-kernel (replaces the ghost fill for them)."""
        check(_lib().lbg_set_periodic_wrap(self.h, (C.c_int * 3)(*[int(bool(w)) for w in wrap])))

    def set_streaming(self, mode):
        """lbg.STREAM_AB (two buffers, default) or lbg.STREAM_AA (in-place, one buffer)."""
        check(_lib().lbg_set_streaming(self.h, int(mode)))

    def stream_only(self, box: CellBox):
        bx = box.c()
        check(_lib().lbg_stream(self.h, C.byref(bx)))

    def fill_periodic(self, periodic, full=True):
        check(_lib().lbg_fill_periodic(self.h, (C.c_int * 3)(*[int(bool(p)) for p in periodic]), int(full)))

    def apply_boundaries(self, spec: BcSpec, touches):
        check(_lib().lbg_apply_boundaries(self.h, spec.c(), (C.c_int * 6)(*[int(bool(t)) for t in touches])))

    def map(self, snaps, subdivisions=8):
        arr, n = snapshot_array(snaps)
        check(_lib().lbg_map(self.h, arr, n, subdivisions))

    def map_prepare(self, snaps, subdivisions=8):
        """Map into the shadow fraction field (the current one stays in use)."""
        arr, n = snapshot_array(snaps)
        check(_lib().lbg_map_prepare(self.h, arr, n, subdivisions))

    def map_commit(self):
        check(_lib().lbg_map_commit(self.h))

    def set_force_mode(self, mode):
        """lbg.FORCE_SCRATCH (reference scratch + finalize) or lbg.FORCE_FUSED (the PSM
        kernel sums per-particle force/torque with warp aggregation + atomics)."""
        check(_lib().lbg_set_force_mode(self.h, int(mode)))

    def set_solid_velocities(self, snaps):
        arr, n = snapshot_array(snaps)
        check(_lib().lbg_set_solid_velocities(self.h, arr, n))

    def reduce_hydro(self, mode=_abi.REDUCE_PARITY, capacity=None):
        cap = capacity or 1 << 16
        out = (_abi.HydroPartial * cap)()
        n = C.c_int()
        check(_lib().lbg_reduce_hydro(self.h, mode, out, cap, C.byref(n)))
        ids = np.array([out[i].id for i in range(n.value)], dtype=np.int32)
        rows = np.zeros((n.value, 12))
        for i in range(n.value):
            rows[i] = list(out[i].f) + list(out[i].f_comp) + list(out[i].t) + list(out[i].t_comp)
        return ids, rows

    # coupling fields
    def _frac_arrays(self):
        nx, ny, nz = self.dims
        shp = (nz, ny, nx)
        return {"count": np.zeros(shp, np.uint8), "id0": np.zeros(shp, np.int32),
                "id1": np.zeros(shp, np.int32), "b0": np.zeros(shp), "b1": np.zeros(shp),
                "btot": np.zeros(shp)}

    def download_fraction(self):
        f = self._frac_arrays()
        check(_lib().lbg_download_fraction(self.h, *[_ptr(f[k]) for k in ("count", "id0", "id1", "b0", "b1", "btot")]))
        return f

    def upload_fraction(self, f):
        arrs = [np.ascontiguousarray(f[k]) for k in ("count", "id0", "id1", "b0", "b1", "btot")]
        check(_lib().lbg_upload_fraction(self.h, *[_ptr(a) for a in arrs]))

    def _vec_pair(self, fn, a=None, b=None, download=False):
        nx, ny, nz = self.dims
        if download:
            a, b = np.zeros((nz, ny, nx, 3)), np.zeros((nz, ny, nx, 3))
            check(fn(self.h, _ptr(a), _ptr(b)))
            return a, b
        # None leaves that side untouched (a null pointer at the C ABI)
        a = None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        b = None if b is None else np.ascontiguousarray(b, dtype=np.float64)
        check(fn(self.h, None if a is None else _ptr(a), None if b is None else _ptr(b)))

    def download_solid_velocity(self):
        return self._vec_pair(_lib().lbg_download_solid_velocity, download=True)

    def upload_solid_velocity(self, v0, v1):
        self._vec_pair(_lib().lbg_upload_solid_velocity, v0, v1)

    def download_scratch(self):
        return self._vec_pair(_lib().lbg_download_scratch, download=True)

    def upload_scratch(self, m0, m1):
        self._vec_pair(_lib().lbg_upload_scratch, m0, m1)

    # barrier / observers
    def sync(self) -> dict:
        e = _abi.Errors()
        check(_lib().lbg_sync(self.h, C.byref(e)))
        return {"unstable": e.unstable_cells, "overfull": e.overfull_cells, "unknown": e.unknown_ids}

    def total_mass(self) -> float:
        v = C.c_double()
        check(_lib().lbg_total_mass(self.h, C.byref(v)))
        return v.value

    def total_momentum(self):
        v = (C.c_double * 3)()
        check(_lib().lbg_total_momentum(self.h, v))
        return np.array(list(v))

    def observe(self, f_ext=(0.0, 0.0, 0.0)) -> dict:
        """Fluid part of io::sample_scalars (output.cpp:22-45) as one device reduction."""
        out = (C.c_double * 6)()
        check(_lib().lbg_observe(self.h, (C.c_double * 3)(*f_ext), out))
        v = list(out)
        return {"mass": v[0], "momentum": np.array(v[1:4]), "fluid_ke": v[4], "max_u": v[5]}

    def moments(self, with_frac=False) -> np.ndarray:
        """Per-cell {rho, mx, my, mz[, btot]} of the src interior, shape (nz, ny, nx, 4|5):
        the reference's own per-cell sums (lbm.cpp:61-93), for observers and grid dumps."""
        nx, ny, nz = self.dims
        S = 5 if with_frac else 4
        out = np.empty((nz, ny, nx, S), dtype=np.float64)
        check(_lib().lbg_moments(self.h, 1 if with_frac else 0, out.ctypes.data))
        return out

    # halo
    def comm_init(self, nranks, rank, uid: bytes, axis=2, periodic=(1, 1, 1)):
        check(_lib().lbg_comm_init(self.h, nranks, rank, uid, axis,
                                   (C.c_int * 3)(*[int(bool(p)) for p in periodic])))

    # fused P2P halo (lbg_p2p.cu)
    def p2p_handles(self) -> bytes:
        buf = C.create_string_buffer(256)
        n = C.c_size_t()
        check(_lib().lbg_p2p_handles(self.h, buf, C.byref(n)))
        return buf.raw[: n.value]

    def p2p_connect(self, nranks, rank, all_handles: bytes, axis=2, periodic=(1, 1, 1)):
        check(_lib().lbg_p2p_connect(self.h, nranks, rank, all_handles, axis,
                                     (C.c_int * 3)(*[int(bool(p)) for p in periodic])))

    def p2p_prime(self):
        check(_lib().lbg_p2p_prime(self.h))

    def sweep_outer_p2p(self, params: FluidParams):
        fl = params.c()
        check(_lib().lbg_sweep_outer_p2p(self.h, C.byref(fl)))

    def halo_begin(self):
        check(_lib().lbg_halo_begin(self.h))

    def halo_complete(self):
        check(_lib().lbg_halo_complete(self.h))

    # instrumentation
    def halo_stage(self, offsets):
        """begin_halo_exchange (sim.cpp:156-179) without the host: stage source_slab(o) of every
        neighbour offset on the device."""
        flat = [int(v) for o in offsets for v in o]
        check(_lib().lbg_halo_stage(self.h, (C.c_int * max(1, len(flat)))(*flat), len(offsets)))

    def halo_fetch(self, direction, src: "Block"):
        """complete_halo_exchange for one neighbour entry: src's staged source_slab(-dir) into
        this block's ghost_region(dir), device to device."""
        check(_lib().lbg_halo_fetch(self.h, (C.c_int * 3)(*direction), src.h))

    def halo_fetch_all(self, entries):
        """complete_halo_exchange for all (direction, source Block) entries in one launch."""
        n = len(entries)
        dirs = (C.c_int * (3 * max(n, 1)))(*[v for d, _ in entries for v in d])
        srcs = (C.c_void_p * max(n, 1))(*[s.h.value for _, s in entries])
        check(_lib().lbg_halo_fetch_all(self.h, dirs, srcs, n))

    def halo_push_connect(self, entries):
        """entries: [(offset (ox, oy, oz), Block)] — the neighbours this block pushes into."""
        n = len(entries)
        offs = (C.c_int * (3 * max(n, 1)))(*[v for o, _ in entries for v in o])
        blks = (C.c_void_p * max(n, 1))(*[b.h.value for _, b in entries])
        check(_lib().lbg_halo_push_connect(self.h, offs, blks, n))

    def halo_push(self):
        check(_lib().lbg_halo_push(self.h))

    def halo_push_wait(self):
        check(_lib().lbg_halo_push_wait(self.h))

    def set_timing(self, on=True):
        check(_lib().lbg_set_timing(self.h, int(on)))

    def timings(self):
        ms = (C.c_double * 8)()
        n = (C.c_longlong * 8)()
        check(_lib().lbg_timings(self.h, ms, n))
        return {_abi.CATEGORIES[i]: (ms[i], n[i]) for i in range(8)}


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(_lib().lbg_comm_unique_id(buf))
    return buf.raw


def launch_count() -> int:
    return int(_lib().lbg_launch_count())


# --------------------------------------------------------------------------- operator API
def collide_stream(block: Block, params: FluidParams, box: CellBox) -> None:
    """lbm::collide_stream_{serial,omp} (lbm.cpp:53-59): fused pull + SRT over `box`;
    raises NumericError after the sweep if any cell tripped the stability guard."""
    params.validate()
    block.sweep(params, box)
    block.sync()


psm_collide_stream = collide_stream  # psm.cpp:266-276 — the block's coupling flag selects PSM


def fill_periodic_ghosts(block: Block, periodic) -> None:
    """lbm::fill_periodic_ghosts (boundary.cpp:98-137), all 19 q of all 26 regions."""
    block.fill_periodic(periodic, full=True)
    block.sync()


def apply_boundaries(block: Block, spec: BcSpec, touches) -> None:
    """lbm::apply_boundaries (boundary.cpp:140-146)."""
    block.apply_boundaries(spec, touches)
    block.sync()


def build_fraction_field(block: Block, snapshots, subdivisions: int = 8) -> None:
    """SubBlockRegistry::build + psm::build_fraction_field (psm.cpp:55-136). The solid
    velocities (psm.cpp:138-169) follow from these snapshots until set_solid_velocities
    registers a new list; the PSM kernels evaluate them inline. NumericError if a cell sees
    more than two particles."""
    block.map(snapshots, subdivisions)
    block.sync()


def set_solid_velocities(block: Block, snapshots) -> None:
    """psm::set_solid_velocities (psm.cpp:138-169); SyncError on unknown ids."""
    block.set_solid_velocities(snapshots)
    block.sync()


def finalize_hydro_forces(block: Block, mode: int = _abi.REDUCE_PARITY) -> list[HydroPartial]:
    """psm::finalize_hydro_forces (psm.cpp:278-322): id-sorted partials, clears the scratch."""
    ids, rows = block.reduce_hydro(mode)
    return [HydroPartial(int(i), r[0:3].copy(), r[3:6].copy(), r[6:9].copy(), r[9:12].copy())
            for i, r in zip(ids, rows)]
