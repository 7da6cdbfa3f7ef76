"""CPU ORACLE for the Serinv hot path (arXiv 2503.17528) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import or execute anything under oracle/.  The product
path (paper_2503_17528_b200/, libserinv.so) never imports, links or calls it,
and shares no code with it (no kernels, helpers, tables or constants).

What it computes (plain, slow, obviously correct; float64; numpy/scipy library
primitives -- Cholesky, triangular solve, matmul, dense inverse -- serve as
steps, with no blocking, fusion or reordering beyond the paper's listings):

  dense.py       the plain definitions: dense expansion of a BTA matrix, the
                 dense Cholesky factor / dense inverse restricted to the BTA
                 pattern, log det.
  sequential.py  POBTAF (Alg. 1), POBTASI (Alg. 2),
                 log det = 2 sum log diag(L).
  parallel.py    partition plan (Sec. 3.1), PARTIAL_/PERMUTED_POBTAF
                 (Alg. 3-4), reduced system + POBTARSSI (Sec. 3.3,
                 P:509-518), PARTIAL_/PERMUTED_POBTASI (Alg. 5-6),
                 and the in-process P-partition pipeline PSELINV.
  closed_form.py the G2K Kronecker closed form of the selected inverse and
                 log det (pin at full scale).
  invariants.py  L L^T = A on the pattern; (X A) restricted to pattern-only
                 products = I; per-block relative Frobenius errors.

Pins (tests/test_oracle_*.py, run with -m "not gpu"): numpy.linalg dense
Cholesky / inverse / slogdet of the N x N expansion, closed forms, the
parallel == sequential equivalence, Fig. 2's n=11, P=3 partition,
n_r = 2P-1, invariants, and mutation sensitivity.  Parity status of
each function is listed in DESIGN.md ("Oracle pins").  Every function here is
pinned; none is "parity unpinned".
"""
