"""Fluid-step driver over liblbg: slab decomposition + the GPU fluid phases of
Simulation::step (sim.cpp:269-338) for one block per GPU.

* ``SlabDecomposition`` is partition::decompose (partition.cpp:27-83) restricted to a 1-D
  block grid along one axis — {1,1,N} z-slabs for configs 2/4, {N,1,1} x-slabs for config 5 —
  with the halo protocol liblbg's NCCL exchange implements (lbg_halo.cu): per step each rank
  sends its first plane's inbound-to-prev populations to ``prev`` and its last plane's
  inbound-to-next populations to ``next``, posted in the fixed order
  (send next, recv prev, send prev, recv next) so the two messages of a rank pair match even
  when prev == next.
* ``FluidStepper`` issues one fluid step: [halo begin] -> inner sweep -> [halo complete] ->
  boundary fill -> outer sweep -> swap, with the periodic axes the block spans wrapped
  in-kernel and the others filled by the halo / BC kernels, exactly the order of
  phase_post_and_map / phase_setu_inner / phase_outer_reduce.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import lbdem

Q_AXIS = {  # q with c_axis = +1 / -1, lattice.hpp:18-29
    0: ((1, 7, 9, 11, 13), (2, 8, 10, 12, 14)),
    1: ((3, 7, 10, 15, 17), (4, 8, 9, 16, 18)),
    2: ((5, 11, 14, 15, 18), (6, 12, 13, 16, 17)),
}


@dataclass
class SlabDecomposition:
    domain: tuple
    nranks: int
    axis: int = 2
    periodic: tuple = (1, 1, 1)

    def __post_init__(self):
        d = self.domain[self.axis]
        if d % self.nranks:
            raise lbdem.ConfigError(
                f"block grid does not divide the domain evenly in axis {self.axis} "
                f"({d} / {self.nranks})")  # partition.cpp:31-34
        self.ext = d // self.nranks

    def block_dims(self) -> tuple:
        dims = list(self.domain)
        dims[self.axis] = self.ext
        return tuple(dims)

    def block_lo(self, rank: int) -> tuple:
        lo = [0, 0, 0]
        lo[self.axis] = rank * self.ext
        return tuple(lo)

    def prev(self, rank: int) -> int:
        if rank > 0:
            return rank - 1
        return self.nranks - 1 if self.periodic[self.axis] else -1

    def next(self, rank: int) -> int:
        if rank < self.nranks - 1:
            return rank + 1
        return 0 if self.periodic[self.axis] else -1

    def domain_faces(self, rank: int) -> tuple:
        """BlockInfo::domain_faces (partition.cpp:57-60)."""
        t = [True] * 6
        t[2 * self.axis] = rank == 0
        t[2 * self.axis + 1] = rank == self.nranks - 1
        return tuple(t)

    def wrap_axes(self) -> tuple:
        """Periodic axes a single block spans: wrapped in-kernel (lbg_set_periodic_wrap)."""
        return tuple(int(bool(self.periodic[a]) and (a != self.axis or self.nranks == 1)) for a in range(3))

    def posting_order(self, rank: int) -> list:
        """(op, peer, buffer) in the order lbg_halo_begin posts them."""
        out = []
        if self.next(rank) >= 0:
            out.append(("send", self.next(rank), "hi"))
        if self.prev(rank) >= 0:
            out.append(("recv", self.prev(rank), "lo"))
        if self.prev(rank) >= 0:
            out.append(("send", self.prev(rank), "lo"))
        if self.next(rank) >= 0:
            out.append(("recv", self.next(rank), "hi"))
        return out


class FluidStepper:
    """GPU fluid phases of one block (sim.cpp:269-338), one block per GPU."""

    def __init__(self, decomp: SlabDecomposition, rank: int, params: lbdem.FluidParams,
                 bc: lbdem.BcSpec | None = None, coupling: bool = False, device: int = 0,
                 uid: bytes | None = None, halo: str = "nccl", allgather=None):
        """halo: "nccl" (pack -> ncclSend/Recv on the comm stream -> unpack, hidden behind
        the inner sweep) or "p2p" (the outer sweep stores the outbound populations straight
        into the neighbours' ghost planes over NVLink; plain fluid, >= 2 ranks). For "p2p",
        `allgather(bytes) -> list[bytes]` exchanges the CUDA IPC handles in rank order."""
        self.decomp, self.rank, self.params = decomp, rank, params
        self.halo = halo
        self.bc = bc or lbdem.BcSpec()
        self.bc.validate()
        params.validate()
        dims = decomp.block_dims()
        self.block = lbdem.Block(dims, lo=decomp.block_lo(rank), coupling=coupling, device=device)
        self.touches = decomp.domain_faces(rank)
        self.has_bc = any(self.touches[f] and self.bc.faces[f].kind != lbdem.BcKind.periodic for f in range(6))
        # In-kernel wrap is exact only when no wall ring meets the wrapped axis: a wall face
        # writes its edge ghosts with its own formula (boundary.cpp:99-133), which a wrapped
        # pull would bypass. With walls, periodic axes go through the ghost fill instead.
        self.wrap = decomp.wrap_axes() if not self.has_bc else (0, 0, 0)
        self.fill = tuple(0 if self.has_bc is False else w for w in decomp.wrap_axes())
        self.block.set_periodic_wrap(self.wrap)
        self.exchange = decomp.nranks > 1 or (decomp.periodic[decomp.axis] and not decomp.wrap_axes()[decomp.axis])
        self.p2p = halo == "p2p" and decomp.nranks > 1
        if self.p2p:
            if coupling or self.has_bc:
                raise lbdem.ConfigError("the P2P halo is the plain periodic-fluid path")
            handles = allgather(self.block.p2p_handles())
            self.block.p2p_connect(decomp.nranks, rank, b"".join(handles), axis=decomp.axis,
                                   periodic=decomp.periodic)
        elif self.exchange:
            self.block.comm_init(decomp.nranks, rank, uid or b"\0" * 128, axis=decomp.axis,
                                 periodic=decomp.periodic)
        a = decomp.axis
        n = dims[a]
        lo, hi = [0, 0, 0], list(dims)
        lo[a], hi[a] = 1, n - 1
        self.inner = lbdem.CellBox(tuple(lo), tuple(hi))
        outer = []
        for plane in (0, n - 1) if n > 1 else (0,):
            blo, bhi = [0, 0, 0], list(dims)
            blo[a], bhi[a] = plane, plane + 1
            outer.append(lbdem.CellBox(tuple(blo), tuple(bhi)))
        self.outer = outer
        self.full = lbdem.CellBox((0, 0, 0), dims)

    def prime(self) -> None:
        """P2P mode: fill the slab-axis ghost planes once from the neighbours (call after
        every rank set its state and passed a host barrier)."""
        if self.p2p:
            self.block.p2p_prime()

    def step(self) -> None:
        b = self.block
        if self.p2p:
            b.sweep(self.params, self.inner)
            b.sweep_outer_p2p(self.params)
            b.swap()
            return
        if not self.exchange and not self.has_bc:
            b.sweep(self.params, self.full)
        else:
            if self.exchange:
                b.halo_begin()
            if not self.has_bc:
                b.sweep(self.params, self.inner)  # needs no ghost of the slab axis
            if self.exchange:
                b.halo_complete()
            if self.has_bc:
                if any(self.fill):
                    b.fill_periodic(self.fill, full=False)
                b.apply_boundaries(self.bc, self.touches)
                b.sweep(self.params, self.full)
            else:
                b.sweep_boxes(self.params, self.outer)
        b.swap()
