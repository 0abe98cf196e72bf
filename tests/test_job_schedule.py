"""CPU check of the streamed host job's schedule (paper_2303_11811_b200/csrc/lbg_job_schedule.hpp,
the op sequence lbg_run_host enqueues) against the double-buffer semantics: every sweep reads
step s-1 values (wrap or NCCL seam across z), every (step, plane) computed once, every plane
uploaded before use and downloaded once holding the final step, no write to a plane already
queued for download — for 20,000 (nz, steps, slab, seam) cases (tests/cpp/job_schedule_check.cpp)."""
import os
import subprocess

from conftest import ROOT


def test_streamed_job_schedule_is_hazard_free(tmp_path):
    exe = tmp_path / "job_schedule_check"
    subprocess.check_call(["g++", "-O2", "-std=c++17", f"-I{os.path.join(ROOT, 'paper_2303_11811_b200', 'csrc')}",
                           os.path.join(ROOT, "tests", "cpp", "job_schedule_check.cpp"), "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), (r.returncode, r.stdout, r.stderr)
