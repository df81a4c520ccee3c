"""LoKA hot-path ORACLE — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU (numpy float64) definitions of what the
FP8 linear+norm hot path computes, written from
PAPER.md (arXiv 2605.10886) and, where the paper is silent, from the readings
listed in DESIGN.md §"Readings".  Every function cites the passage it follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2605_10886_b200``) never imports it, and this package never imports
the product path: the two share no code (only ``synth`` input generators,
which hold none of the method's arithmetic).

Parity pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function here
to something other than itself: closed forms, library routines (torch CPU FP8
casts, cuda_fp8.hpp host casts, numpy BLAS, torch float64 norms), SPEC/paper
worked values (tests/golden/), and brute force on tiny inputs.  The paper
prints no worked numeric example for any of these steps, so no function's
parity is pinned to a number printed in the paper except the Table II
geomean fixture.
"""
from . import fp8, quantize, linear, probe, dispatch, track, sample, nvfp4, gradcomm  # noqa: F401
