"""The coupled-sweep parity tests under every selectable kernel variant (the switches are read
once per process, so each variant runs the tests in a subprocess):
  LBG_K12=2 / 3 the unified coupled sweep / the covered-list split always (the default picks one
  per block by its covered fraction); LBG_K12_PIPE=0 the unified coupled sweep without the
  register pipeline (LBG_K12_SM=4/6 its
  occupancy caps), LBG_K12_TWO=0 two-entry segments in their own kernel, LBG_K12_NOWRAP=0 the
  generic pull for unwrapped blocks;
  LBG_K12=0 the K1 || K2 split instead of the unified coupled sweep, with LBG_K2_MODE=0 plain
  segment loop, 1 register-pipelined (split default), 2 TMA-fed one-entry K2, LBG_K2_CONCURRENT=0
  K2 after K1 on one stream; LBG_DIRECT_INDEX=0 solid velocities through id0 -> id table;
  LBG_SWEEP_PAIR=1 the 128-bit K1;
  LBDEM_GPU_SWEEP=split the drop-in in the reference's inner / halo / BC / outer-shell order;
  LBDEM_GPU_PREMAP=1 the next step's mapping prepared during the last DEM sub-cycle;
  LBDEM_GPU_HALO=stage the staged 19-q device halo instead of the pushed one; LBG_WALK_ROWS=1 /
  LBG_WALK_REGS=120 the force reduction's row walk / register cap; LBG_MAP_COL=0 the level-outer
  mapping kernel (LBG_MAP_MINB=5: at 48 registers), LBG_MAP_CTA_WARPS=4 the column mapping kernel
  in CTAs of 4 warps; LBDEM_GPU_FAST_SYNC=0 the drop-in's host particle messaging exactly as the
  reference writes it; LBG_K12_TMA=1 the TMA-fed unified coupled sweep."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SELECT = "coupled or setu or fused or mapping_and_solid or shear or sweep or finalize or hydro"
DROPIN = "config1_known_answers or particle_bed or decomposition_invariance or config5_layout_scratch"


@pytest.mark.parametrize("env", [{"LBG_K12": "2"}, {"LBG_K12": "3"}, {"LBG_K12_PIPE": "0"}, {"LBG_K12_TWO": "0"},
                                 {"LBG_K12_NOWRAP": "0"},
                                 {"LBG_K12": "0"}, {"LBG_K12": "0", "LBG_K2_MODE": "0"},
                                 {"LBG_K12": "0", "LBG_K2_MODE": "2"}, {"LBG_K12": "0", "LBG_K2_CONCURRENT": "0"},
                                 {"LBG_DIRECT_INDEX": "0"}, {"LBG_K12_PIPE": "0", "LBG_K12_SM": "4"},
                                 {"LBG_K12_PIPE": "0", "LBG_K12_SM": "6"},
                                 {"LBG_SWEEP_PAIR": "1"}, {"LBDEM_GPU_SWEEP": "split"}, {"LBDEM_GPU_PREMAP": "1"},
                                 {"LBDEM_GPU_HALO": "stage"}, {"LBG_WALK_ROWS": "1"}, {"LBG_WALK_REGS": "120"},
                                 {"LBG_MAP_COL": "0"}, {"LBG_MAP_COL": "0", "LBG_MAP_MINB": "5"},
                                 {"LBG_MAP_CTA_WARPS": "4"}, {"LBDEM_GPU_FAST_SYNC": "0"},
                                 {"LBG_K12_TMA": "1"}, {"LBG_K12_TMA": "1", "LBG_K12": "2"}],
                         ids=lambda env: "-".join(f"{k}_{v}" for k, v in env.items()))
def test_parity_suite_under_variant(env):
    e = dict(os.environ, **env)
    # the parity cases, and drop-in runs vs the reference (config 1: periodic block, in-kernel
    # wrap; the bed: walls, inflow, outflow; 2x2x2 decomposition)
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(ROOT, "tests", "test_gpu_parity.py"),
                        os.path.join(ROOT, "tests", "test_dropin.py"), "-m", "gpu", "-q", "-x",
                        "-k", f"({SELECT}) or {DROPIN}", "-p", "no:cacheprovider"],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    tail = (r.stdout + r.stderr)[-2000:]
    assert r.returncode == 0, tail
    assert " passed" in tail and "failed" not in tail, tail
