"""ctypes front end of the drop-in build (integration/_build/liblbdem_dropin.so): the
reference Simulation whose GPU-side operators run on liblbg. Same row formats as
oracle/pyoracle.RefSim so tests compare the two runs directly."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "liblbdem_dropin.so")


class DropinError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def load(path: str = SO):
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built (python integration/make_dropin.py)")
        L = C.CDLL(path)
        vp = C.c_void_p
        dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
        L.dropin_last_error.restype = C.c_char_p
        L.dropin_sim_create.restype = vp
        L.dropin_sim_create.argtypes = [C.c_char_p]
        L.dropin_sim_destroy.argtypes = [vp]
        L.dropin_sim_run.argtypes = [vp, C.c_long]
        L.dropin_sim_add_particles.argtypes = [vp, C.c_int, dp]
        L.dropin_sim_cells.restype = C.c_long
        L.dropin_sim_cells.argtypes = [vp]
        L.dropin_sim_num_particles.restype = C.c_int
        L.dropin_sim_num_particles.argtypes = [vp]
        L.dropin_sim_particles.argtypes = [vp, dp]
        L.dropin_sim_pdfs.argtypes = [vp, dp]
        L.dropin_sim_mass.restype = C.c_double
        L.dropin_sim_mass.argtypes = [vp]
        L.dropin_sim_shear_wave.argtypes = [vp]
        L.dropin_sim_reset_timers.argtypes = [vp]
        L.dropin_sim_timings.argtypes = [vp, dp]
        L.dropin_sim_observe.argtypes = [vp, dp]
        L.dropin_sim_grid_dump.argtypes = [vp, C.c_char_p]
        _lib = L
    return _lib


class DropinSim:
    def __init__(self, cfg_json: str, domain):
        self.L = load()
        self.h = self.L.dropin_sim_create(cfg_json.encode())
        if not self.h:
            raise DropinError(-1, self.L.dropin_last_error().decode())
        self.domain = tuple(domain)

    def close(self):
        if getattr(self, "h", None):
            self.L.dropin_sim_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc:
            raise DropinError(rc, self.L.dropin_last_error().decode())

    def run(self, steps):
        self._check(self.L.dropin_sim_run(self.h, steps))

    def add_particles(self, rows):
        """rows: (n, 6) of id, x, y, z, r, m (Simulation::add_particles)"""
        rows = np.ascontiguousarray(rows, dtype=np.float64)
        self._check(self.L.dropin_sim_add_particles(self.h, len(rows), rows))

    def shear_wave(self):
        self._check(self.L.dropin_sim_shear_wave(self.h))

    def pdfs(self):
        nx, ny, nz = self.domain
        a = np.zeros((nz, ny, nx, 19))
        self.L.dropin_sim_pdfs(self.h, a)
        return a

    def particles(self):
        n = self.L.dropin_sim_num_particles(self.h)
        rows = np.zeros((max(n, 1), 16))
        if n:
            self.L.dropin_sim_particles(self.h, rows)
        return rows[:n]

    def mass(self):
        return self.L.dropin_sim_mass(self.h)

    def observe(self):
        """io::sample_scalars: [step, mass, px, py, pz, fluid_ke, particle_ke, min_gap, max_u]."""
        out = np.zeros(9)
        self._check(self.L.dropin_sim_observe(self.h, out))
        return out

    def grid_dump(self, path):
        self._check(self.L.dropin_sim_grid_dump(self.h, str(path).encode()))

    def reset_timers(self):
        self.L.dropin_sim_reset_timers(self.h)

    def timings(self):
        out = np.zeros(8)
        self.L.dropin_sim_timings(self.h, out)
        return out
