"""CPU oracle for the FD block preconditioner of Montardini, Sangalli & Tani (arXiv:1712.00403).

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package. The
product path (``paper_1712_00403_b200``) never imports, links or executes anything here,
and this package never imports the product path: the two share no code. The only shared
module is ``synth`` (seeded inputs, no method arithmetic).

Plain, slow, obviously correct: FP64 numpy/scipy, each function citing the PAPER.md passage
(``P:line``) it follows. Library primitives (matmul, tensordot, LAPACK ``eigh``, banded
Cholesky) serve as single steps; there is no blocking, fusion or reordering beyond the
paper's algorithm. Readings of ambiguous passages are SURVEY.md §8(c) C-1..C-20, listed in
DESIGN.md.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to something other than
itself: closed forms, invariants, brute-force dense solves and brute-force 3D quadrature.
Parity status per function is listed in DESIGN.md §"Oracle pins"; nothing is unpinned.
"""
from . import splines, univariate, kron, fd, mass, spaces, precond  # noqa: F401
