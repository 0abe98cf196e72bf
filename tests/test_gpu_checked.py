"""The GPU suites again on the CHECKED build of liblbg (make checked -> build_checked/liblbg.so,
-DLBG_CHECKED): every computed buffer index in the sweep, mapping, reduction, boundary and halo
kernels is range-checked, and every sweep verifies that it wrote each cell of its box exactly
once across all of its kernels (the unified coupled sweep || the two-entry kernel, K1 || K2 on
two streams, TMA-fed K2, shell sweeps, the pipelined and plain unified sweeps with two-entry
segments inline or in their own kernel) and nothing outside. lbg_sync turns a violation into an
error, so any out-of-range index or double/missing write fails the suite. This is the
repository's memcheck/racecheck (compute-sanitizer is closed on the GPU pool). The library is
the same sources; LBG_LIB points the ctypes binding at it and LD_LIBRARY_PATH the drop-in."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

CHECKED = os.path.join(ROOT, "paper_2303_11811_b200", "build_checked", "liblbg.so")


def _run(files, extra_env=None, k=None):
    if not os.path.exists(CHECKED):
        pytest.fail("checked build missing: make -C paper_2303_11811_b200 checked")
    env = dict(os.environ, LBG_LIB=CHECKED,
               LD_LIBRARY_PATH=os.path.dirname(CHECKED) + ":" + os.environ.get("LD_LIBRARY_PATH", ""),
               LBG_EXPECT_CHECKED="1", **(extra_env or {}))
    cmd = [sys.executable, "-m", "pytest", *[os.path.join(ROOT, "tests", f) for f in files], "-m", "gpu", "-q",
           "-x", "-p", "no:cacheprovider"]
    if k:
        cmd += ["-k", k]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=3000)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail


def test_checked_library_is_loaded():
    """Inside the checked runs: the ctypes binding and the drop-in use build_checked/liblbg.so."""
    if os.environ.get("LBG_EXPECT_CHECKED") != "1":
        pytest.skip("runs inside the checked subprocesses")
    from paper_2303_11811_b200 import lbg
    assert b"checked" in lbg.load().lbg_version()
    maps = open("/proc/self/maps").read()
    assert "build_checked/liblbg.so" in maps


def test_dropin_uses_checked_library():
    """Inside the checked runs: the drop-in's liblbg dependency resolves to the checked build."""
    if os.environ.get("LBG_EXPECT_CHECKED") != "1":
        pytest.skip("runs inside the checked subprocesses")
    sys.path.insert(0, os.path.join(ROOT, "integration"))
    import dropin
    dropin.load()
    maps = open("/proc/self/maps").read()
    assert "build_checked/liblbg.so" in maps
    assert "paper_2303_11811_b200/liblbg.so" not in maps


SELF = "not suites_checked and not variants_checked"


def test_parity_suites_checked():
    _run(["test_gpu_checked.py", "test_gpu_parity.py", "test_gpu_aa.py", "test_gpu_reference_cases.py", "test_gpu_job.py"],
         k=SELF)


def test_dropin_suites_checked():
    _run(["test_gpu_checked.py", "test_dropin.py", "test_gpu_multi.py"], k=SELF)


@pytest.mark.parametrize("env", [{"LBG_K12": "2"}, {"LBG_K12": "3"}, {"LBG_K12_PIPE": "0"}, {"LBG_K12_TWO": "0"},
                                 {"LBG_K12": "0"}, {"LBG_K12": "0", "LBG_K2_MODE": "2"},
                                 {"LBG_K12": "0", "LBG_K2_CONCURRENT": "0"}, {"LBG_SWEEP_PAIR": "1"}])
def test_sweep_variants_checked(env):
    _run(["test_gpu_parity.py", "test_dropin.py"], extra_env=env,
         k="coupled or setu or fused or sweep or shear or particle_bed or decomposition_invariance")
