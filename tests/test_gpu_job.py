"""GPU parity of the streamed host job (lbg_run_host: upload, sweeps and download pipelined over
z-slabs) against the step-by-step C-ABI path and the CPU oracle.

The bar is bitwise: interior cells after K steps equal those of lbg_upload_src + K x (whole-block
lbg_sweep + lbg_swap) + lbg_download_src (and of K oracle steps, fill_periodic + collide_stream,
sim.cpp:702-704 / lbm.cpp:21-49); ghost cells keep their input values.
"""
import ctypes as C

import numpy as np
import pytest

from conftest import equal_bits, interior, n_bit_mismatch, random_pdf

pytestmark = pytest.mark.gpu

ALL_P = (1, 1, 1)


def stepwise(gpu, dims, src0, params, steps):
    blk = gpu.Block(dims)
    blk.set_periodic_wrap(ALL_P)
    blk.upload_src(src0)
    for _ in range(steps):
        blk.sweep(params, gpu.CellBox((0, 0, 0), dims))
        blk.swap()
    blk.sync()
    out = blk.download_src()
    blk.close()
    return out


def pinned_copy(gpu, a):
    """a copy of `a` in pinned host memory (lbg_host_alloc); returns (array, pointer)."""
    from paper_2303_11811_b200 import lbg as abi
    p = C.c_void_p()
    gpu.check(abi.load().lbg_host_alloc(a.nbytes, C.byref(p)))
    h = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=a.shape)
    h[...] = a
    return h, p


def free_pinned(p):
    from paper_2303_11811_b200 import lbg as abi
    abi.load().lbg_host_free(p)


@pytest.mark.parametrize("dims,steps,slab,fext", [
    ((16, 12, 40), 5, 4, (0.0, 0.0, 0.0)),     # several slabs, cone narrower than the domain
    ((16, 12, 40), 6, 0, (1e-5, 0.0, -2e-5)),  # default slab (16 planes), forced
    ((13, 7, 9), 1, 1, (0.0, 0.0, 0.0)),       # one-plane slabs, odd step count
    ((8, 8, 5), 9, 2, (2e-6, 1e-6, 0.0)),      # more steps than planes: everything in the tail
    ((33, 5, 24), 0, 5, (0.0, 0.0, 0.0)),      # no steps: a round trip
    ((40, 9, 17), 4, 17, (0.0, 0.0, 0.0)),     # one slab: the tail only
])
def test_run_host_matches_stepwise(gpu, dims, steps, slab, fext):
    src0 = random_pdf(dims, seed=11 + steps)
    params = gpu.FluidParams(0.8, fext)
    want = stepwise(gpu, dims, src0, params, steps)
    host, p = pinned_copy(gpu, src0)
    try:
        blk = gpu.Block(dims)
        blk.set_periodic_wrap(ALL_P)
        errs = blk.run_host(params, host, steps, slab)
        assert errs["unstable"] == 0
        got = host.copy()
        assert n_bit_mismatch(interior(got), interior(want)) == 0
        # ghost cells keep their input values
        g = np.ones(src0.shape, bool)
        g[:, 1:-1, 1:-1, 1:-1] = False
        assert np.array_equal(got[g].view(np.uint64), src0[g].view(np.uint64))
        # the block's src holds the final state afterwards
        assert equal_bits(interior(blk.download_src()), interior(want))
        blk.close()
    finally:
        free_pinned(p)


@pytest.mark.parametrize("steps,slab", [(5, 4), (9, 2), (3, 40)])
def test_run_host_z_seam_through_the_halo(gpu, steps, slab):
    """z not wrapped in-kernel but the slab axis of an NCCL halo (one rank: the periodic
    self-exchange): the seam planes take one halo exchange per step; bitwise the wrapped job"""
    dims = (12, 10, 40)
    src0 = random_pdf(dims, seed=8)
    params = gpu.FluidParams(0.75, (0.0, 2e-6, 0.0))
    want = stepwise(gpu, dims, src0, params, steps)
    blk = gpu.Block(dims)
    blk.set_periodic_wrap((1, 1, 0))
    blk.comm_init(1, 0, b"\0" * 128, axis=2, periodic=ALL_P)
    host = src0.copy()
    blk.run_host(params, host, steps, slab)
    assert n_bit_mismatch(interior(host), interior(want)) == 0
    blk.close()


def test_run_host_matches_oracle(gpu, oracle):
    dims, steps, tau, fext = (12, 10, 21), 4, 0.7, (1e-5, -1e-5, 0.0)
    src0 = random_pdf(dims, seed=5)
    a = src0.copy()
    for _ in range(steps):
        oracle.fill_periodic(dims, a, ALL_P)
        d = np.zeros_like(a)
        assert oracle.collide_stream(dims, a, d, tau, fext, (0, 0, 0), dims) == 0
        a = d
    host = src0.copy()  # pageable host memory works too (copies do not overlap then)
    blk = gpu.Block(dims)
    blk.set_periodic_wrap(ALL_P)
    blk.run_host(gpu.FluidParams(tau, fext), host, steps, 3)
    assert n_bit_mismatch(interior(host), interior(a)) == 0
    blk.close()


def test_run_host_twice_and_after_steps(gpu):
    """the job starts from the host field, not the block's state, and may be repeated"""
    dims = (16, 8, 20)
    params = gpu.FluidParams(0.9)
    src0 = random_pdf(dims, seed=2)
    want = stepwise(gpu, dims, src0, params, 6)
    blk = gpu.Block(dims)
    blk.set_periodic_wrap(ALL_P)
    blk.fill_equilibrium(1.0, (0.01, 0.0, 0.0))
    blk.sweep(params, gpu.CellBox((0, 0, 0), dims))
    blk.swap()
    host = src0.copy()
    blk.run_host(params, host, 3, 4)
    blk.run_host(params, host, 3, 7)
    assert n_bit_mismatch(interior(host), interior(want)) == 0
    blk.close()


def test_run_host_rejects_unsupported_blocks(gpu):
    dims = (8, 8, 8)
    host = random_pdf(dims, seed=1)
    params = gpu.FluidParams(0.8)
    blk = gpu.Block(dims)
    with pytest.raises(Exception, match="periodic"):
        blk.run_host(params, host, 1)  # no in-kernel wrap
    blk.set_periodic_wrap(ALL_P)
    with pytest.raises(gpu.ConfigError):
        blk.run_host(gpu.FluidParams(0.5), host, 1)
    blk.close()
    cb = gpu.Block(dims, coupling=True)
    cb.set_periodic_wrap(ALL_P)
    with pytest.raises(Exception, match="plain-fluid"):
        cb.run_host(params, host, 1)
    cb.close()


def test_run_host_reports_unstable_cells(gpu):
    dims = (8, 8, 12)
    host = random_pdf(dims, seed=4)
    host[1, 5, 4, 4] = 50.0  # a cell moving far above the stability limit (lbm.hpp:106)
    blk = gpu.Block(dims)
    blk.set_periodic_wrap(ALL_P)
    with pytest.raises(gpu.NumericError):
        blk.run_host(gpu.FluidParams(0.8), host, 2, 3)
    blk.close()
