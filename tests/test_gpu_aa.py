"""AA-pattern in-place streaming (lbg_set_streaming(LBG_STREAM_AA), lbg_aa.cu) against the
double-buffered pull sweep and the oracle: bitwise equal populations after every step count
(both AA phases: the odd-step state is un-streamed for the download), forced and unforced,
odd extents (rows that end mid-warp, x-wrap at both ends), switching layouts mid-run, the
released buffer, and the operations an AA block refuses."""
import numpy as np
import pytest

from conftest import equal_bits, interior, random_pdf

pytestmark = pytest.mark.gpu

ALL_P = (1, 1, 1)


def _ab_run(gpu, dims, src0, p, steps):
    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.set_periodic_wrap(ALL_P)
    out = []
    for _ in range(steps):
        blk.sweep(p, gpu.CellBox((0, 0, 0), dims))
        blk.swap()
        out.append(interior(blk.download_src()).copy())
    blk.sync()
    blk.close()
    return out


@pytest.mark.parametrize("dims,fext", [((16, 12, 10), (0.0, 0.0, 0.0)),
                                       ((33, 9, 7), (1e-5, 0.0, -2e-5)),
                                       ((64, 5, 3), (0.0, 3e-6, 0.0))])
def test_aa_matches_double_buffer_every_step(gpu, oracle, dims, fext):
    from paper_2303_11811_b200 import lbg
    src0 = random_pdf(dims, seed=41)
    p = gpu.FluidParams(0.8, fext)
    ref = _ab_run(gpu, dims, src0, p, 5)
    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.set_periodic_wrap(ALL_P)
    blk.set_streaming(lbg.STREAM_AA)
    for s in range(5):
        blk.sweep(p, gpu.CellBox((0, 0, 0), dims))
        blk.swap()
        got = interior(blk.download_src())
        assert equal_bits(got, ref[s]), f"step {s + 1}"
    assert blk.sync()["unstable"] == 0
    # the oracle's first step too (pull from periodically filled ghosts)
    o = src0.copy()
    oracle.fill_periodic(dims, o, ALL_P)
    d = np.zeros_like(o)
    oracle.collide_stream(dims, o, d, 0.8, fext, (0, 0, 0), dims)
    assert equal_bits(ref[0], interior(d))


def test_aa_switch_back_mid_run_and_memory(gpu):
    from paper_2303_11811_b200 import lbg
    dims = (24, 10, 6)
    src0 = random_pdf(dims, seed=43)
    p = gpu.FluidParams(0.7)
    ref = _ab_run(gpu, dims, src0, p, 6)
    blk = gpu.Block(dims)
    blk.upload_src(src0)
    blk.set_periodic_wrap(ALL_P)
    import ctypes as C
    L = lbg.load()
    mem = C.c_longlong()
    L.lbg_block_info(blk.h, None, None, None, C.byref(mem))
    before = mem.value
    blk.set_streaming(lbg.STREAM_AA)
    L.lbg_block_info(blk.h, None, None, None, C.byref(mem))
    assert mem.value < before - (before // 3)  # one of the two PDF buffers released
    for _ in range(3):  # odd: the block holds the streamed state S1
        blk.sweep(p, gpu.CellBox((0, 0, 0), dims))
        blk.swap()
    blk.set_streaming(lbg.STREAM_AB)  # S1 -> the double-buffer src
    assert equal_bits(interior(blk.download_src()), ref[2])
    for _ in range(3):
        blk.sweep(p, gpu.CellBox((0, 0, 0), dims))
        blk.swap()
    assert equal_bits(interior(blk.download_src()), ref[5])


def test_aa_refusals(gpu):
    from paper_2303_11811_b200 import lbg
    dims = (16, 8, 8)
    blk = gpu.Block(dims)
    blk.fill_equilibrium(1.0, (0.0, 0.0, 0.0))
    with pytest.raises(Exception):
        blk.set_streaming(lbg.STREAM_AA)
        blk.sweep(gpu.FluidParams(0.8), gpu.CellBox((0, 0, 0), dims))  # no wrap: refused
    blk.set_periodic_wrap(ALL_P)
    with pytest.raises(Exception):
        blk.sweep(gpu.FluidParams(0.8), gpu.CellBox((0, 0, 0), (8, 8, 8)))  # sub-box
    with pytest.raises(Exception):
        blk.download_dst()
    with pytest.raises(Exception):
        blk.fill_periodic(ALL_P)
    blk.sweep(gpu.FluidParams(0.8), gpu.CellBox((0, 0, 0), dims))
    blk.swap()
    with pytest.raises(Exception):
        blk.total_mass()  # odd step: moments need the S0 state
    blk.sweep(gpu.FluidParams(0.8), gpu.CellBox((0, 0, 0), dims))
    blk.swap()
    assert abs(blk.total_mass() - 16 * 8 * 8) < 1e-9
    cb = gpu.Block(dims, coupling=True)
    with pytest.raises(Exception):
        cb.set_streaming(lbg.STREAM_AA)
