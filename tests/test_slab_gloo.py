"""World-size-2 CPU test (gloo) of the slab halo protocol liblbg's NCCL exchange implements
(lbg_halo.cu, paper_2303_11811_b200/driver.py::SlabDecomposition): two ranks each own a
z-slab of a periodic domain, exchange the 5 inbound populations of their boundary planes in
the fixed posting order, wrap the received planes' rings along x/y, sweep with the oracle,
and the union equals the single-domain oracle step bitwise (the reference's decomposition
invariance, acceptance criterion 11)."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT, random_pdf


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, domain, axis, out_q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle.pyoracle import Oracle
    from paper_2303_11811_b200.driver import Q_AXIS, SlabDecomposition

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    dec = SlabDecomposition(domain, world, axis=axis, periodic=(1, 1, 1))
    dims = dec.block_dims()
    lo = dec.block_lo(rank)
    glob = random_pdf(domain, seed=123, ghosts=False)  # same on every rank
    # this rank's block, reference layout [q, k, j, i] with ghosts
    sl = [slice(None)] * 4
    for a in range(3):
        ax = 3 - a  # array axis of coordinate a
        sl[ax] = slice(1 + lo[a], 1 + lo[a] + dims[a])
    blk = np.zeros((19, dims[2] + 2, dims[1] + 2, dims[0] + 2))
    blk[:, 1:-1, 1:-1, 1:-1] = glob[tuple(sl)]

    up, dn = Q_AXIS[axis]
    ax = 3 - axis  # array axis of the slab axis

    def plane(arr, idx, qs):
        s = [list(qs)] + [slice(1, -1)] * 3
        s[ax] = idx
        return np.ascontiguousarray(arr[tuple(s)])

    send = {"hi": torch.from_numpy(plane(blk, dims[axis], up)),  # last interior plane (index n)
            "lo": torch.from_numpy(plane(blk, 1, dn))}
    recv = {"lo": torch.zeros_like(send["hi"]), "hi": torch.zeros_like(send["lo"])}
    reqs = []
    for op, peer, buf in dec.posting_order(rank):
        reqs.append(dist.isend(send[buf], peer) if op == "send" else dist.irecv(recv[buf], peer))
    for r in reqs:
        r.wait()

    def put(arr, idx, qs, vals):
        s = [list(qs)] + [slice(1, -1)] * 3
        s[ax] = idx
        arr[tuple(s)] = vals

    put(blk, 0, up, recv["lo"].numpy())
    put(blk, dims[axis] + 1, dn, recv["hi"].numpy())
    # ring wrap of the received planes along the face axes + local periodic fill of the
    # face axes (regions without a slab-axis offset)
    per = [1, 1, 1]
    per[axis] = 0
    orc.fill_periodic(dims, blk, per)
    for gidx in (0, dims[axis] + 1):
        sel = [slice(None)] * 4
        sel[ax] = gidx
        pl = blk[tuple(sel)]  # [q, b, a] plane incl. its ring
        pl[:, 0, :] = pl[:, -2, :]
        pl[:, -1, :] = pl[:, 1, :]
        pl[:, :, 0] = pl[:, :, -2]
        pl[:, :, -1] = pl[:, :, 1]
    dst = np.zeros_like(blk)
    bad = orc.collide_stream(dims, blk, dst, 0.8, (1e-6, 0.0, -1e-6), (0, 0, 0), dims)
    gathered = [torch.zeros_like(torch.from_numpy(dst)) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(dst))
    if rank == 0:
        full = np.zeros_like(glob)
        for r in range(world):
            lo_r = dec.block_lo(r)
            s = [slice(None)] * 4
            for a in range(3):
                s[3 - a] = slice(1 + lo_r[a], 1 + lo_r[a] + dims[a])
            full[tuple(s)] = gathered[r].numpy()[:, 1:-1, 1:-1, 1:-1]
        g = glob.copy()
        orc.fill_periodic(domain, g, (1, 1, 1))
        gd = np.zeros_like(g)
        orc.collide_stream(domain, g, gd, 0.8, (1e-6, 0.0, -1e-6), (0, 0, 0), domain)
        same = np.array_equal(full[:, 1:-1, 1:-1, 1:-1].view(np.uint64), gd[:, 1:-1, 1:-1, 1:-1].view(np.uint64))
        out_q.put((same, bad))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,domain,axis", [(2, (6, 5, 8), 2), (2, (8, 4, 5), 0), (3, (5, 4, 9), 2),
                                               (8, (4, 3, 16), 2)])  # the 8-GPU ring of config 4
def test_slab_halo_protocol_gloo(world, domain, axis):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, domain, axis, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs)
    same, bad = q.get(timeout=5)
    assert bad == 0
    assert same


def test_decomposition_rules():
    from paper_2303_11811_b200 import lbdem
    from paper_2303_11811_b200.driver import SlabDecomposition
    d = SlabDecomposition((512, 512, 2048), 4)
    assert d.block_dims() == (512, 512, 512)
    assert [d.prev(r) for r in range(4)] == [3, 0, 1, 2]
    assert [d.next(r) for r in range(4)] == [1, 2, 3, 0]
    assert d.wrap_axes() == (1, 1, 0)
    d8 = SlabDecomposition((512, 512, 4096), 8)  # config 4 at 8 GPUs
    assert d8.block_dims() == (512, 512, 512) and d8.block_lo(7) == (0, 0, 3584)
    assert [d8.prev(r) for r in range(8)] == [7, 0, 1, 2, 3, 4, 5, 6]
    assert d.domain_faces(0) == (True, True, True, True, True, False)
    nd = SlabDecomposition((64, 32, 32), 2, axis=0, periodic=(0, 1, 1))
    assert nd.prev(0) == -1 and nd.next(1) == -1
    assert nd.posting_order(0) == [("send", 1, "hi"), ("recv", 1, "hi")]
    assert SlabDecomposition((8, 8, 8), 1).wrap_axes() == (1, 1, 1)
    with pytest.raises(lbdem.ConfigError):
        SlabDecomposition((8, 8, 9), 2)
