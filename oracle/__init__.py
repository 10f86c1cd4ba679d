"""CPU oracle for the B200 hot path — TEST INFRASTRUCTURE ONLY.

A NumPy/SciPy restatement of the reference algorithms (`sgkkt`, mounted at
/root/reference/pkg/src/sgkkt, a pure-Python package: there is nothing to
compile, so there is no oracle/_ref).  Each function cites the reference
file:line it follows.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package, and only as the
checker or the timed CPU baseline — never on the product path.

Pinning: tests/test_oracle_golden.py checks every function here against
golden vectors produced by the reference itself (tests/golden/make_golden.py,
run in the build container where /root/reference exists).  The CG / MINRES
drivers, the Legendre triple products, the separable KL expansion, the
unit-square domain and the forward-problem load vector have no reference
implementation: those are pinned against independent oracles (SciPy CG
iteration counts, dense direct solves, Gauss-Legendre quadrature) and are
marked "parity unpinned (no reference implementation)" in DESIGN.md.
"""

from .sgk_oracle import *  # noqa: F401,F403
