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
