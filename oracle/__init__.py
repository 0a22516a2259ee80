"""CPU oracle for the blocked randomized QB factorization of Martinsson & Voronin
(arXiv 1503.07157), "randQB_b" / "randQB_pb" (Fig. 2, and Fig. 4,
lines 859-887).

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import it.  The product
path (``paper_1503_07157_b200``) never imports, calls or links anything under ``oracle/``,
and the oracle never imports the product package: the two share no code.

Contents
--------
``omega``   counter-based Philox4x32-10 Gaussian generator for Ω, numpy.
``qb``      the algorithm itself, step by step in the paper's order and notation, FP64 numpy;
            ``orth`` is a packaged economy QR exactly as the paper defines it.

Pins (tests/test_oracle_*.py, run with ``-m "not gpu"``) tie every function to something
other than itself: Random123 known-answer vectors, libm/mpmath accuracy bounds, the
paper's relations (Proposition 1 at :538-543), Eckart-Young (:229-239),
the blocked == unblocked projector theorem (:631-648), the power-scheme identity
(:805-810), SPEC.md worked examples, and brute-force SVD on tiny inputs.  Functions with no
such pin are marked "parity unpinned" in their docstring and in DESIGN.md §6.
"""
from . import omega, qb  # noqa: F401
