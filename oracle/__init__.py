"""TEST INFRASTRUCTURE — parity checkers for the B200 path (never imported by the product).

* ``oracle.pyoracle.Oracle`` — ctypes/numpy front end of ``liboracle.so``, the plain-C
  restatement of the reference operators (``lbm_oracle.c``).
* ``oracle.pyoracle.RefLib`` — ctypes front end of ``_ref/liblbdem_ref.so``, the unmodified
  reference sources compiled by ``oracle/Makefile`` with ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this package.
"""
