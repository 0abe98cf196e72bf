"""Multi-GPU slab decomposition with the NCCL halo (K7), bitwise against the single-domain
oracle. Needs >= 2 GPUs (gpurun --gpus 2/4); skipped on one."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpus():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("axis,halo", [(2, "nccl"), (0, "nccl"), (2, "p2p"), (0, "p2p")])
def test_slab_halo_bitwise(axis, halo):
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    env = dict(os.environ, SLAB_AXIS=str(axis), SLAB_STEPS="4", SLAB_HALO=halo)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={min(n, 4)}", "--master-addr=127.0.0.1",
                        "--master-port=29531", os.path.join(HERE, "mp_halo_gpu.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.parametrize("halo", ["nccl", "p2p"])
def test_streamed_job_z_slabs_bitwise(halo):
    """lbg_run_host on every rank's z-slab (upload, sweeps, download pipelined over 3-plane
    slabs; the seam planes take one NCCL halo exchange per step) against the single-domain
    oracle: bitwise."""
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    env = dict(os.environ, SLAB_AXIS="2", SLAB_STEPS="5", SLAB_HALO=halo, SLAB_JOB="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        f"--nproc-per-node={min(n, 4)}", "--master-addr=127.0.0.1",
                        "--master-port=29537", os.path.join(HERE, "mp_halo_gpu.py")],
                       env=env, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0


@pytest.mark.parametrize("halo", ["p2p", "nccl"])
def test_config4_full_size_two_gpus_vs_one_block(halo):
    """Config 4 at 512^3 per GPU on 2 GPUs against the same 512 x 512 x 1024 domain as one
    block: per-plane hashes of the per-cell moments equal over all 2.7e8 cells (tests/
    mp_fullsize_gpu.py). Needs 131 GB on GPU 0."""
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    env = dict(os.environ, SLAB_HALO=halo, SLAB_STEPS="3")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(HERE, "mp_fullsize_gpu.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    assert "rank 1: 0 of 512 z-planes differ" in r.stdout


@pytest.mark.parametrize("halo,per", [("push", 1), ("stage", 1), ("host", 1), ("push", 2), ("push", 4)])
def test_dropin_bed_spread_over_gpus_bitwise(halo, per, monkeypatch):
    """The drop-in with its blocks dealt over the GPUs (LBDEM_GPU_SPREAD=1: `per` consecutive
    blocks per GPU, one worker thread per block): a config-3-shaped bed on {N*per,1,1} x-slabs
    (N = 2..4; per = 4 is config 5's layout) with host DEM, the PDF halo pushed by each sender
    after its sweep (5 q per face cell, NVLink peer stores between GPUs, device stores between
    slabs of one GPU), or staged 19-q slabs, or host slabs; PARITY force partials — every PDF
    and particle state bitwise equal to the CPU reference."""
    n = _ngpus()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    import torch  # noqa: F401  (CUDA plumbing)
    sys.path.insert(0, os.path.join(os.path.dirname(HERE), "integration"))
    import dropin
    from conftest import equal_bits
    from oracle.pyoracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    g = min(n, 4)
    monkeypatch.setenv("LBDEM_GPU_SPREAD", "1")
    monkeypatch.setenv("LBDEM_GPU_HALO", halo)
    monkeypatch.setenv("LBDEM_GPU_BLOCKS_PER_DEVICE", str(per))  # consecutive slabs per GPU
    nb = g * per
    cfg = ('{"scenario":"fluidized_bed_dense","domain":[%d,32,48],"blocks":[%d,1,1],"workers":%d,'
           '"particles":{"count":24},"physical":{"diameter_cells":8},'
           '"fluid":{"bc":{"xm":"no_slip","xp":"no_slip","ym":"no_slip","yp":"no_slip",'
           '"zm":"velocity","zp":"pressure"}},'
           '"dem":{"k_n":230,"d_n":520,"k_t":65,"d_t":260,"subcycles":10,"settle_subcycles":20}}'
           % (20 * nb, nb, nb))
    a = dropin.DropinSim(cfg, (20 * nb, 32, 48))
    ref = RefLib()
    ref.set_threads(2)
    b = ref.sim(cfg)
    a.run(5)
    b.run(5)
    assert equal_bits(a.particles(), b.particles())
    assert equal_bits(a.pdfs(), b.pdfs())
