"""Generates tests/golden/* from the REFERENCE ITSELF (oracle/_ref/liblbdem_ref.so, the
unmodified /root/reference sources). Run in the build container:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures pin the plain-C oracle (tests/test_oracle.py) on machines where the reference
sources are absent (the GPU box). Inputs are seeded, outputs are the reference's.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from conftest import random_pdf  # noqa: E402
from oracle.pyoracle import RefLib, fnv1a64, make_snapshots  # noqa: E402

CONFIG1 = ('{"scenario":"settling_sphere","domain":[64,64,64],"particles":{"count":1},'
           '"physical":{"u_gravity":0.06},"dem":{"k_n":230,"d_n":520,"k_t":65,"d_t":260,"subcycles":10}}')


def main():
    ref = RefLib()
    out = {}
    # 1. fused forced sweep on a random periodic 8^3 field (test_lattice_lbm.cpp:251-301)
    dims = (8, 8, 8)
    src = random_pdf(dims, seed=29)
    b = ref.block(dims)
    b.set_src(src)
    b.fill_periodic((1, 1, 1))
    fext = np.array([1e-5, 0.0, -2e-5])
    b.sweep(0.8, fext, (0, 0, 0), dims)
    out.update(sweep_dims=np.array(dims), sweep_src=src, sweep_tau=0.8, sweep_fext=fext,
               sweep_out=b.get_dst()[:, 1:-1, 1:-1, 1:-1].copy())
    # 2. bed boundary fill: no-slip sides, velocity inflow, pressure outflow
    dims = (6, 5, 7)
    src = random_pdf(dims, seed=43)
    kinds = np.array([1, 1, 1, 1, 2, 3])
    uw = np.zeros(18)
    uw[12:15] = (0.0, 0.0, 2.2472e-3)
    rho = np.array([1.0] * 6)
    b = ref.block(dims)
    b.set_src(src)
    b.apply_boundaries(list(kinds), uw, list(rho), [1] * 6)
    out.update(bc_dims=np.array(dims), bc_src=src, bc_kinds=kinds, bc_uwall=uw, bc_rho=rho,
               bc_out=b.get_src())
    # 3. two overlapping moving spheres: mapping, setU, PSM step, partials
    dims = (24, 20, 22)
    centers = np.array([(8.3, 10.2, 11.1), (15.6, 9.7, 10.9)])
    radii = np.array([5.0, 4.5])
    fr = np.array([ref.f_of_r(r) for r in radii])
    u = np.array([(0.004, -0.001, 0.002), (-0.003, 0.0, 0.001)])
    w = np.array([(0.0, 0.0005, -0.0002), (0.0003, 0.0, 0.0)])
    snaps = make_snapshots([3, 7], centers, radii, fr, u, w)
    src = random_pdf(dims, seed=77)
    b = ref.block(dims)
    b.set_snapshots(snaps)
    b.map()
    b.set_u()
    f = b.get_fraction()
    b.set_src(src)
    b.fill_periodic((1, 1, 1))
    b.sweep(0.7, (0.0, 0.0, 0.0), (0, 0, 0), dims, coupling=True)
    ids, rows = b.finalize(2)
    out.update(map_dims=np.array(dims), map_ids=np.array([3, 7], np.int32), map_x=centers, map_r=radii,
               map_fr=fr, map_u=u, map_w=w, map_src=src, map_tau=0.7, map_count=f["count"],
               map_btot=f["btot"], map_out=b.get_dst()[:, 1:-1, 1:-1, 1:-1].copy(),
               map_partial_ids=ids, map_partials=rows)
    # large arrays are stored as FNV-1a hashes; inputs are regenerated from their seeds
    small = {}
    for k, v in out.items():
        v = np.asarray(v)
        if k.endswith("_src"):
            continue
        if v.size > 64:
            small[k + "_fnv"] = hex(fnv1a64(np.ascontiguousarray(v)))
        else:
            small[k] = v.tolist()
    small["seeds"] = {"sweep_src": 29, "bc_src": 43, "map_src": 77}
    json.dump(small, open(os.path.join(HERE, "golden.json"), "w"), indent=1)

    # 4. config-1 known answers (re-derived from the reference)
    sim = ref.sim(CONFIG1)
    ka = {"config": CONFIG1, "generator": "oracle/_ref via tests/golden/make_golden.py", "steps": {}}
    done = 0
    for n in (1, 10, 100):
        sim.run(n - done)
        done = n
        p = sim.particles()[0]
        ka["steps"][str(n)] = {"pdf_hash": hex(fnv1a64(sim.pdfs())), "x_z": p[3], "u_z": p[6],
                               "f_hydro": list(p[10:13]), "t_hydro": list(p[13:16]),
                               "f_hydro_z": p[12], "mass": sim.mass()}
    json.dump(ka, open(os.path.join(HERE, "config1_known_answers.json"), "w"), indent=1)
    print(json.dumps(ka["steps"]["10"]), json.dumps(ka["steps"]["100"]))


if __name__ == "__main__":
    main()
