"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what the B200 hot path
computes, written from PAPER.md (arXiv:1604.07994).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import, call, link or execute anything under ``oracle/``.
The product path (``paper_1604_07994_b200``) never does; it shares no code
with this package (only the seeded input generators in ``synth/``).

Modules
-------
``fem``   element matrices by textbook P1 integration on each tetrahedron and
          element-by-element global assembly (scipy CSR) of A (three forms),
          B, C and M; apply; load vectors; gauge; direct solve.
``mg``    the Uzawa-smoothed V_var multigrid of P:1236-1243 written out with
          assembled matrices (transfers from the coarse P1 basis evaluated at
          fine vertices, coloured smoothers, dense coarse solve).
``capi``  ctypes wrapper of ``oracle/c/oracle.c``: the same element-loop apply
          in plain C (OpenMP over cube layers), for sizes scipy cannot hold
          and for the timed CPU baseline.
"""
