"""CPU check of the drop-in's phase scheduler (integration/dropin_sched.hpp) against the
reference ThreadPoolScheduler's contract (partition.hpp:170-192): compiled with the
reference headers, so it runs where /root/reference is present."""
import os
import subprocess

import pytest

from conftest import ROOT

REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_spin_phase_scheduler_keeps_the_thread_pool_contract(tmp_path):
    exe = tmp_path / "sched_check"
    subprocess.check_call(["g++", "-O2", "-std=c++20", "-pthread", f"-I{REF_INC}",
                           f"-I{os.path.join(ROOT, 'integration')}",
                           os.path.join(ROOT, "tests", "cpp", "sched_check.cpp"), "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.returncode, r.stdout, r.stderr)
