"""ORACLE -- test infrastructure, NOT part of the product.

A plain, slow, obviously-correct CPU implementation of what the hot path of
arXiv:1705.08019 (ParaExp + Leapfrog for FIT-discretised Maxwell) computes:
FIT coefficients, the leapfrog iteration, the polynomial exp(tA)v (Newton form on
Leja points / truncated Taylor) and the ParaExp superposition with
staggered reconstruction.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import, call, link or execute anything under
``oracle/``.  It shares no code with ``paper_1705_08019_b200`` (the CUDA path) and
imports nothing from it; the only common module is ``synth`` (seeded inputs, no
method arithmetic).

Pinned by tests/test_oracle_*.py against values the paper/mathematics fix (closed
forms, invariants, dense eigendecompositions, brute force).  Functions without
such a pin say "parity unpinned" in their docstring.
"""
