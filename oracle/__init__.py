"""CPU oracle for the bfsht apply path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package, and only as the checker or the timed CPU reference;
the product (paper_2004_11346_b200) never routes through it.

``oracle.apply`` restates the reference apply algorithm in numpy/scipy
(each function cites the reference file:line it follows); ``oracle.dense``
holds the dense O(N^2)-per-order references.  The oracle is pinned against
the reference's own outputs by tests/test_oracle_golden.py, using the
golden vectors in tests/golden/ written by tests/golden/make_golden.py from
the reference package itself.
"""
