"""CPU checks of the drop-in boundary: liblbg.so loads without a GPU and exports every
function include/lbg.h declares; the host mirror's value types follow the reference."""
import ctypes
import os

import pytest

from paper_2303_11811_b200 import lbdem, lbg


def test_header_declares_the_operator_api():
    syms = lbg.header_symbols()
    for name in ("lbg_block_create", "lbg_sweep", "lbg_sweep_boxes", "lbg_fill_periodic",
                 "lbg_apply_boundaries", "lbg_map", "lbg_set_solid_velocities", "lbg_reduce_hydro",
                 "lbg_halo_begin", "lbg_halo_complete", "lbg_sync", "lbg_comm_init"):
        assert name in syms
    assert len(syms) >= 40


def test_library_exports_every_header_symbol():
    lib = lbg.load()
    missing = [s for s in lbg.header_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_struct_layouts_match_header():
    assert ctypes.sizeof(lbg.Snapshot) == 8 + 8 * 11
    assert ctypes.sizeof(lbg.HydroPartial) == 8 + 8 * 12
    assert ctypes.sizeof(lbg.FaceBc) == 8 + 8 * 4
    assert ctypes.sizeof(lbg.Box) == 24
    assert ctypes.sizeof(lbg.Fluid) == 32


def test_library_is_sm100a_only():
    path = lbg.LIB_PATH
    assert os.path.exists(path)
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_boundary_shell_matches_reference_tiling():
    dims = (7, 6, 5)
    boxes = lbdem.boundary_shell(dims)
    assert len(boxes) == 6
    seen = set()
    for b in boxes:
        for k in range(b.lo[2], b.hi[2]):
            for j in range(b.lo[1], b.hi[1]):
                for i in range(b.lo[0], b.hi[0]):
                    assert (i, j, k) not in seen
                    seen.add((i, j, k))
    shell = {(i, j, k) for k in range(5) for j in range(6) for i in range(7)
             if i in (0, 6) or j in (0, 5) or k in (0, 4)}
    assert seen == shell
    assert lbdem.boundary_shell((2, 5, 5)) == [lbdem.CellBox((0, 0, 0), (2, 5, 5))]


def test_host_validation_mirrors_reference():
    with pytest.raises(lbdem.ConfigError):
        lbdem.FluidParams(0.4).validate()
    assert abs(lbdem.FluidParams(0.8).nu() - 0.1) < 1e-15
    spec = lbdem.BcSpec()
    spec.faces[2] = lbdem.FaceBc(lbdem.BcKind.no_slip)
    with pytest.raises(lbdem.ConfigError):
        spec.validate()
    with pytest.raises(lbdem.ConfigError):
        lbdem.f_of_r(0.5)


def test_f_of_r_matches_oracle_bitwise(oracle):
    for r in (0.75, 1.0, 2.0, 5.0, 10.0, 50.0):
        assert lbdem.f_of_r(r) == oracle.f_of_r(r)


def test_dropin_library_loads_and_exports_its_api():
    """The drop-in build (the reference Simulation over liblbg, integration/make_dropin.py)
    loads without a GPU and exports the entry points its tests and bench call."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "integration"))
    import dropin
    if not os.path.exists(dropin.SO):
        pytest.skip("drop-in not built (needs /root/reference at build time)")
    lib = dropin.load()
    for name in ("dropin_sim_create", "dropin_sim_run", "dropin_sim_pdfs", "dropin_sim_particles",
                 "dropin_sim_timings", "dropin_sim_observe", "dropin_sim_grid_dump"):
        assert hasattr(lib, name), name


def test_tma_variant_uses_bulk_copies_and_mbarriers():
    """The TMA-fed K2 variant (LBG_K2_MODE=2) compiles to sm_100a bulk copies (UBLKCP) completed
    on shared-memory mbarriers (SYNCS.*): the Blackwell data-movement path, not per-thread loads."""
    import subprocess
    out = subprocess.run(["cuobjdump", "-sass", lbg.LIB_PATH], capture_output=True, text=True).stdout
    start = out.find("psm_seg_tma_kernel")
    assert start >= 0
    body = out[start:out.find("Function :", start + 1)]
    assert "UBLKCP" in body and "SYNCS" in body
