"""CPU check of the pushed halo's selection rule (lbg_push.cu, lbg_halo_push): for a neighbour at
offset o the sender pushes, from its source_slab(o) (sim.cpp:120-135), the populations q with
c_q[d] == o[d] on every axis where o[d] != 0 — 5 per face, 1 per edge, none per corner. The
receiver's pull sweep reads a ghost slot (g, q) only when g + c_q is one of its interior cells;
this test enumerates every such read of a small block, finds the neighbour at offset o whose
ghost region holds the slot (ghost_region, sim.cpp:137-152) and checks that q is in the set that
neighbour pushes toward this block (its offset -o) — i.e. the pushed values are a superset of everything a sweep can read, so
interior results equal the full 19-q exchange."""
import itertools

# lattice.hpp:18-29 (the D3Q19 velocity set, rest first, then opposite pairs)
CX = (0, 1, -1, 0, 0, 0, 0, 1, -1, 1, -1, 1, -1, 1, -1, 0, 0, 0, 0)
CY = (0, 0, 0, 1, -1, 0, 0, 1, -1, -1, 1, 0, 0, 0, 0, 1, -1, 1, -1)
CZ = (0, 0, 0, 0, 0, 1, -1, 0, 0, 0, 0, 1, -1, -1, 1, 1, -1, -1, 1)


def pushed(o):
    return {q for q in range(19)
            if all(o[d] == 0 or (CX[q], CY[q], CZ[q])[d] == o[d] for d in range(3))}


def test_push_sets():
    faces = [o for o in itertools.product((-1, 0, 1), repeat=3) if sum(map(abs, o)) == 1]
    edges = [o for o in itertools.product((-1, 0, 1), repeat=3) if sum(map(abs, o)) == 2]
    corners = [o for o in itertools.product((-1, 0, 1), repeat=3) if sum(map(abs, o)) == 3]
    assert all(len(pushed(o)) == 5 for o in faces)
    assert all(len(pushed(o)) == 1 for o in edges)
    assert all(len(pushed(o)) == 0 for o in corners)


def test_pushed_slots_cover_every_pull():
    n = (4, 3, 5)
    for i, j, k in itertools.product(*(range(-1, m + 1) for m in n)):
        g = (i, j, k)
        o = tuple(-1 if g[d] < 0 else (1 if g[d] >= n[d] else 0) for d in range(3))
        if o == (0, 0, 0):
            continue  # interior cell
        for q in range(19):
            s = (i + CX[q], j + CY[q], k + CZ[q])
            if all(0 <= s[d] < n[d] for d in range(3)):
                # pulled by interior cell s; the ghost g belongs to the neighbour at offset o,
                # for which this block sits at -o: it pushes the populations leaving toward -o
                sender_view = tuple(-v for v in o)
                assert q in pushed(sender_view), (g, q, o)
