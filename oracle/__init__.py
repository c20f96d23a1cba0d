"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.

* ``oracle.port``  — ctypes view of ``lzb_oracle.c``, a plain-C restatement of
  the reference algorithm for regular 2D spacetrees (every function cites the
  reference file:line it follows).
* ``oracle.ref``   — ctypes view of ``_ref/liblazymg_ref.so``: the UNMODIFIED
  reference sources compiled in place by ``oracle/Makefile`` plus the
  ``ref_driver.cpp`` harness. Present only where the reference tree was
  available at build time (it is copied to the GPU box as a built file).
"""
