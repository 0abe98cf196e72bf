import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

W = np.array([12, 2, 2, 2, 2, 2, 2, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1, 1]) / 36.0  # lattice.hpp:32-39


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and liblbg.so")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    lib = RefLib()
    # the reference nests OpenMP inside its block-worker threads; bound the team so
    # multi-worker configs do not oversubscribe many-core hosts (spinning OMP teams)
    lib.set_threads(max(1, min(8, (os.cpu_count() or 2) // 2)))
    return lib


def random_pdf(dims, seed, lo=0.95, span=0.1, ghosts=True):
    """w_q * (lo + span * U[0,1)) per slot, like the reference tests (test_lattice_lbm.cpp:257-265)."""
    nx, ny, nz = dims
    rng = np.random.default_rng(seed)
    a = W[:, None, None, None] * (lo + span * rng.random((19, nz + 2, ny + 2, nx + 2)))
    if not ghosts:
        g = np.ones(a.shape, bool)
        g[:, 1:-1, 1:-1, 1:-1] = False
        a[g] = 0.0
    return np.ascontiguousarray(a)


def interior(a):
    return a[:, 1:-1, 1:-1, 1:-1]


def equal_bits(a, b):
    """Bitwise equality of float64 arrays (NaN payloads included)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def n_bit_mismatch(a, b):
    return int(np.count_nonzero(np.ascontiguousarray(a).view(np.uint64) != np.ascontiguousarray(b).view(np.uint64)))


@pytest.fixture(scope="session")
def gpu():
    """The liblbg operator API; fails loudly (no fallback) when CUDA or the library is missing."""
    import torch  # noqa: F401  (CUDA context owner for the process, plumbing only)
    from paper_2303_11811_b200 import lbdem, lbg
    lib = lbg.load()
    if lib.lbg_device_count() < 1:
        pytest.fail("no CUDA device visible to liblbg")
    return lbdem
