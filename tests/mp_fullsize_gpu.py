"""torchrun helper (2 ranks) for tests/test_gpu_multi.py: config 4 at its benchmarked size —
two 512^3 z-slabs of a 512 x 512 x 1024 periodic shear-wave domain, the product FluidStepper
with the halo fused into the outer sweep (P2P, NVLink) or over NCCL, three steps — against
the same domain as ONE block on GPU 0 (87 GB; the in-kernel periodic wrap, no halo). Every
rank hashes each z-plane of its per-cell moments (rho and bare momentum: the reference's own
per-cell sums, lbm.cpp:61-93, computed on the device from the populations) and rank 0
compares them with the single block's plane by plane: a checksum of checksums over all
2.7e8 cells. Exit code 0 = every plane equal."""
import hashlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def plane_digests(mom):
    return [hashlib.blake2b(mom[k].tobytes(), digest_size=16).digest() for k in range(mom.shape[0])]


def main():
    import torch
    import torch.distributed as dist

    from paper_2303_11811_b200 import lbdem
    from paper_2303_11811_b200.driver import FluidStepper, SlabDecomposition

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    steps = int(os.environ.get("SLAB_STEPS", "3"))
    halo = os.environ.get("SLAB_HALO", "p2p")
    n = int(os.environ.get("SLAB_N", "512"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    domain = (n, n, n * world)
    dec = SlabDecomposition(domain, world, axis=2, periodic=(1, 1, 1))
    uid = [lbdem.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    params = lbdem.FluidParams(0.8)

    def allgather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    st = FluidStepper(dec, rank, params, device=local, uid=uid[0], halo=halo, allgather=allgather)
    st.block.init_shear_wave(domain)
    torch.cuda.synchronize()
    dist.barrier()
    st.prime()
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(steps):
        st.step()
    st.block.sync()
    mine = plane_digests(st.block.moments())
    st.block.close()
    dist.barrier()
    allp = allgather(mine)
    ok = True
    if rank == 0:
        one = lbdem.Block(domain)
        one.set_periodic_wrap((1, 1, 1))
        one.init_shear_wave(domain)
        box = lbdem.CellBox((0, 0, 0), domain)
        for _ in range(steps):
            one.sweep(params, box)
            one.swap()
        one.sync()
        want = plane_digests(one.moments())
        one.close()
        for r in range(world):
            lo = dec.block_lo(r)[2]
            bad = sum(1 for k, d in enumerate(allp[r]) if d != want[lo + k])
            print(f"rank {r}: {bad} of {len(allp[r])} z-planes differ", flush=True)
            ok &= bad == 0
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
