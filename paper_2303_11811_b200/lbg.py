"""ctypes binding of liblbg.so (include/lbg.h) — the C-ABI the reference's FFI would bind.

This module only declares signatures; ``lbdem.py`` mirrors the reference operator API on
top of it. Loading fails loudly when the CUDA library is missing: there is no CPU fallback
on the LBM/PSM path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# LBG_LIB: another build of the same library (the bounds/race-checked build,
# build_checked/liblbg.so from `make checked`); never a different implementation
LIB_PATH = os.environ.get("LBG_LIB") or os.path.join(HERE, "liblbg.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include", "lbg.h")

OK, CONFIG_ERROR, NUMERIC_ERROR, SYNC_ERROR, IO_ERROR, CUDA_ERROR, INVALID = range(7)
BC_PERIODIC, BC_NO_SLIP, BC_VELOCITY, BC_PRESSURE = range(4)
REDUCE_PARITY, REDUCE_FAST = 0, 1
STREAM_AB, STREAM_AA = 0, 1
FORCE_SCRATCH, FORCE_FUSED = 0, 1
CATEGORIES = ("PSM", "PSM-comm", "mapping", "setU", "redF", "PD", "PD-comm", "other")  # perf.hpp:17-26


class Box(C.Structure):  # lbg_box / CellBox
    _fields_ = [("lo", C.c_int * 3), ("hi", C.c_int * 3)]


class Fluid(C.Structure):  # lbg_fluid / FluidParams
    _fields_ = [("tau", C.c_double), ("f_ext", C.c_double * 3)]


class FaceBc(C.Structure):  # lbg_face_bc / FaceBc
    _fields_ = [("kind", C.c_int), ("pad_", C.c_int), ("u_wall", C.c_double * 3), ("rho", C.c_double)]


class Snapshot(C.Structure):  # lbg_snapshot / ParticleSnapshot
    _fields_ = [("id", C.c_int), ("pad_", C.c_int), ("x", C.c_double * 3), ("r", C.c_double),
                ("f_r", C.c_double), ("u", C.c_double * 3), ("omega", C.c_double * 3)]


class HydroPartial(C.Structure):  # lbg_hydro_partial / HydroPartial
    _fields_ = [("id", C.c_int), ("pad_", C.c_int), ("f", C.c_double * 3), ("f_comp", C.c_double * 3),
                ("t", C.c_double * 3), ("t_comp", C.c_double * 3)]


class Errors(C.Structure):  # lbg_errors
    _fields_ = [("unstable_cells", C.c_longlong), ("overfull_cells", C.c_longlong),
                ("unknown_ids", C.c_longlong)]


_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load liblbg.so once (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"liblbg.so not built at {path}; run __graft_entry__.build() "
                           "(there is no CPU fallback for the GPU path)")
    L = C.CDLL(path)
    vp, i3, d3 = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
    blk = C.c_void_p
    st = C.c_int
    sig = {
        "lbg_last_error": (C.c_char_p, []),
        "lbg_version": (C.c_char_p, []),
        "lbg_device_count": (C.c_int, []),
        "lbg_host_alloc": (st, [C.c_size_t, C.POINTER(C.c_void_p)]),
        "lbg_host_free": (st, [vp]),
        "lbg_block_create": (st, [C.c_int, i3, i3, C.c_int, C.POINTER(C.c_void_p)]),
        "lbg_block_destroy": (st, [blk]),
        "lbg_block_info": (st, [blk, i3, i3, C.POINTER(C.c_int), C.POINTER(C.c_longlong)]),
        "lbg_block_stream": (vp, [blk]),
        "lbg_upload_src": (st, [blk, vp]),
        "lbg_download_src": (st, [blk, vp]),
        "lbg_upload_dst": (st, [blk, vp]),
        "lbg_download_dst": (st, [blk, vp]),
        "lbg_fill_equilibrium": (st, [blk, C.c_double, d3]),
        "lbg_fill_ghosts_src": (st, [blk, C.c_double]),
        "lbg_init_shear_wave": (st, [blk, i3]),
        "lbg_swap": (st, [blk]),
        "lbg_run_host": (st, [blk, C.POINTER(Fluid), vp, C.c_int, C.c_int, C.POINTER(Errors)]),
        "lbg_sweep": (st, [blk, C.POINTER(Fluid), C.POINTER(Box)]),
        "lbg_sweep_boxes": (st, [blk, C.POINTER(Fluid), C.POINTER(Box), C.c_int]),
        "lbg_stream": (st, [blk, C.POINTER(Box)]),
        "lbg_set_streaming": (st, [blk, C.c_int]),
        "lbg_set_periodic_wrap": (st, [blk, i3]),
        "lbg_fill_periodic": (st, [blk, i3, C.c_int]),
        "lbg_apply_boundaries": (st, [blk, C.POINTER(FaceBc), i3]),
        "lbg_map": (st, [blk, C.POINTER(Snapshot), C.c_int, C.c_int]),
        "lbg_map_prepare": (st, [blk, C.POINTER(Snapshot), C.c_int, C.c_int]),
        "lbg_map_commit": (st, [blk]),
        "lbg_set_solid_velocities": (st, [blk, C.POINTER(Snapshot), C.c_int]),
        "lbg_set_force_mode": (st, [blk, C.c_int]),
        "lbg_reduce_hydro": (st, [blk, C.c_int, C.POINTER(HydroPartial), C.c_int, C.POINTER(C.c_int)]),
        "lbg_upload_fraction": (st, [blk, vp, vp, vp, vp, vp, vp]),
        "lbg_download_fraction": (st, [blk, vp, vp, vp, vp, vp, vp]),
        "lbg_upload_solid_velocity": (st, [blk, vp, vp]),
        "lbg_download_solid_velocity": (st, [blk, vp, vp]),
        "lbg_upload_scratch": (st, [blk, vp, vp]),
        "lbg_download_scratch": (st, [blk, vp, vp]),
        "lbg_sync": (st, [blk, C.POINTER(Errors)]),
        "lbg_total_mass": (st, [blk, d3]),
        "lbg_total_momentum": (st, [blk, d3]),
        "lbg_observe": (st, [blk, d3, d3]),
        "lbg_moments": (st, [blk, C.c_int, vp]),
        "lbg_comm_unique_id": (st, [C.c_char_p]),
        "lbg_comm_init": (st, [blk, C.c_int, C.c_int, C.c_char_p, C.c_int, i3]),
        "lbg_comm_destroy": (st, [blk]),
        "lbg_halo_begin": (st, [blk]),
        "lbg_halo_complete": (st, [blk]),
        "lbg_pack_slab": (st, [blk, i3, vp, C.c_longlong, C.POINTER(C.c_longlong)]),
        "lbg_unpack_slab": (st, [blk, i3, vp, C.c_longlong]),
        "lbg_halo_stage": (st, [blk, i3, C.c_int]),
        "lbg_halo_fetch": (st, [blk, i3, blk]),
        "lbg_halo_fetch_all": (st, [blk, i3, C.POINTER(C.c_void_p), C.c_int]),
        "lbg_halo_push_connect": (st, [blk, i3, C.POINTER(C.c_void_p), C.c_int]),
        "lbg_halo_push": (st, [blk]),
        "lbg_halo_push_wait": (st, [blk]),
        "lbg_p2p_handles": (st, [blk, vp, C.POINTER(C.c_size_t)]),
        "lbg_p2p_connect": (st, [blk, C.c_int, C.c_int, C.c_char_p, C.c_int, i3]),
        "lbg_p2p_prime": (st, [blk]),
        "lbg_sweep_outer_p2p": (st, [blk, C.POINTER(Fluid)]),
        "lbg_p2p_destroy": (st, [blk]),
        "lbg_set_timing": (st, [blk, C.c_int]),
        "lbg_timings": (st, [blk, d3, C.POINTER(C.c_longlong)]),
        "lbg_launch_count": (C.c_longlong, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def header_symbols(path: str = INCLUDE) -> list[str]:
    """Every function declared in include/lbg.h (for the export test)."""
    import re
    text = open(path).read()
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(lbg_\w+)\s*\(", text, flags=re.M)))
