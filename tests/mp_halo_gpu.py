"""torchrun helper for tests/test_gpu_multi.py: N ranks (one GPU each) run the product
FluidStepper (z- or x-slabs, NCCL halo hidden behind the inner sweep) for a few steps on a
seeded random periodic field; rank 0 gathers the slabs and compares with the single-domain
oracle bitwise. Exit code 0 = bitwise equal."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    import torch
    import torch.distributed as dist

    from conftest import random_pdf
    from oracle.pyoracle import Oracle
    from paper_2303_11811_b200 import lbdem
    from paper_2303_11811_b200.driver import FluidStepper, SlabDecomposition

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    axis = int(os.environ.get("SLAB_AXIS", "2"))
    steps = int(os.environ.get("SLAB_STEPS", "3"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    domain = [24, 20, 18]
    domain[axis] = 8 * world
    domain = tuple(domain)
    dec = SlabDecomposition(domain, world, axis=axis, periodic=(1, 1, 1))
    uid = [lbdem.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    params = lbdem.FluidParams(0.7, (1e-6, -2e-6, 0.0))
    halo = os.environ.get("SLAB_HALO", "nccl")

    def allgather(b: bytes):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    st = FluidStepper(dec, rank, params, device=local, uid=uid[0], halo=halo, allgather=allgather)
    dims, lo = dec.block_dims(), dec.block_lo(rank)
    glob = random_pdf(domain, seed=321, ghosts=False)
    sl = [slice(None)] * 4
    for a in range(3):
        sl[3 - a] = slice(1 + lo[a], 1 + lo[a] + dims[a])
    mine = np.zeros((19, dims[2] + 2, dims[1] + 2, dims[0] + 2))
    mine[:, 1:-1, 1:-1, 1:-1] = glob[tuple(sl)]
    if os.environ.get("SLAB_JOB") == "1":
        # the streamed host job (lbg_run_host) on each rank's host slab; its seam planes take
        # the NCCL halo (a P2P-mode stepper gets an NCCL comm for it)
        if st.p2p:
            st.block.comm_init(world, rank, uid[0], axis=2, periodic=(1, 1, 1))
        host = mine.copy()
        dist.barrier()
        st.block.run_host(params, host, steps, int(os.environ.get("SLAB_JOB_PLANES", "3")))
        res = torch.from_numpy(np.ascontiguousarray(host[:, 1:-1, 1:-1, 1:-1])).cuda()
    else:
        st.block.upload_src(mine)
        dist.barrier()
        st.prime()
        torch.cuda.synchronize()
        dist.barrier()
        for _ in range(steps):
            st.step()
        st.block.sync()
        res = torch.from_numpy(np.ascontiguousarray(st.block.download_src()[:, 1:-1, 1:-1, 1:-1])).cuda()
    parts = [torch.zeros_like(res) for _ in range(world)]
    dist.all_gather(parts, res)
    ok = True
    if rank == 0:
        orc = Oracle()
        g = glob.copy()
        for _ in range(steps):
            orc.fill_periodic(domain, g, (1, 1, 1))
            d = np.zeros_like(g)
            orc.collide_stream(domain, g, d, 0.7, (1e-6, -2e-6, 0.0), (0, 0, 0), domain)
            g = d
        for r in range(world):
            lo_r = dec.block_lo(r)
            s = [slice(None)] * 4
            for a in range(3):
                s[3 - a] = slice(lo_r[a], lo_r[a] + dims[a])
            want = np.ascontiguousarray(g[:, 1:-1, 1:-1, 1:-1][tuple(s)])
            got = parts[r].cpu().numpy()
            bad = int(np.count_nonzero(got.view(np.uint64) != want.view(np.uint64)))
            print(f"rank {r}: {bad} mismatching slots", flush=True)
            ok &= bad == 0
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
