"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU (numpy, float64) implementation of what the
ParaDiag hot path of Garai & Mandal (arXiv 2304.14021, /root/reference/PAPER.md)
computes.  Every function cites the passage it follows ("P:L" = PAPER.md line L).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2304_14021_b200``) never imports it and shares no code with it; the only
shared module is ``workloads`` (seeded input generators, no method arithmetic).

Readings of the paper where it is silent / ambiguous are listed in DESIGN.md §3
and referenced here as "R#n".

Pins: every module is pinned by ``tests/test_oracle_*.py`` against closed forms,
dense brute force, library eigensolvers or values printed in the paper.  No
function here is "parity unpinned" except where its docstring says so.
"""
from . import spatial, circulant, precond, iterate, sequential, modespace, theory, diagnostics  # noqa: F401
