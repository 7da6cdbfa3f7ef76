"""Pins for oracle/sequential.py (POBTAF Alg. 1, POBTASI Alg. 2) -- CPU only.

Each check compares the block recurrences with something other than themselves:
the numpy.linalg dense Cholesky / inverse / slogdet of the N x N expansion
("L is the Cholesky factor", "true inverse blocks"), and the
size-independent invariants L L^T = A, (X A)|pattern = I.
"""
import numpy as np
import pytest

import btagen
from oracle import dense, invariants as inv, sequential as seq

TOL_L = 1e-11
TOL_X = 1e-11


def _check(A):
    L, X, ld = seq.selinv(A)
    eL, wL = inv.max_block_err(L, dense.dense_cholesky_pattern(A))
    eX, wX = inv.max_block_err(X, dense.dense_inverse_pattern(A))
    ldd = dense.dense_logdet(A)
    assert eL < TOL_L, (eL, wL)
    assert eX < TOL_X, (eX, wX)
    assert abs(ld - ldd) <= 1e-12 * max(1.0, abs(ldd))
    assert inv.llt_residual(L, A) < 1e-12
    assert inv.xa_residual(X, A) < 1e-13
    # strict upper triangle of diagonal factors is zero; X_ii symmetric
    for i in range(A["diag"].shape[0]):
        assert np.all(np.triu(L["diag"][i], 1) == 0.0)
        np.testing.assert_allclose(X["diag"][i], X["diag"][i].T, rtol=0, atol=1e-13 * np.abs(X["diag"][i]).max())
    return L, X, ld


@pytest.mark.parametrize("gen", ["g1", "g2", "g2k"])
def test_c1_against_dense(gen):
    # BASELINE configs[0]: tiny BTA n=8, b=4, a=2 checked against dense Cholesky/inverse
    for seed in range(1, 21):
        _check(btagen.generate(gen, seed, 8, 4, 2))


def test_property_sweep():
    # SPEC S:543 idea: random shapes n in [1,12], b in [1,9], a in [0,5]
    rng = np.random.default_rng(12345)
    for t in range(60):
        n = int(rng.integers(1, 13))
        b = int(rng.integers(1, 10))
        a = int(rng.integers(0, 6))
        gen = ["g1", "g2", "g2k"][t % 3]
        _check(btagen.generate(gen, 100 + t, n, b, a))


def test_bt_special_case_a0():
    # a BT matrix is BTA with a = 0
    L, X, ld = _check(btagen.g1(7, 6, 5, 0))
    assert X["tip"].shape == (0, 0)


def test_single_block():
    _check(btagen.g2(3, 1, 6, 3))


def test_identity():
    n, b, a = 4, 3, 2
    A = dict(diag=np.array([np.eye(b)] * n), lower=np.zeros((n - 1, b, b)),
             arrow=np.zeros((n, a, b)), tip=np.eye(a))
    L, X, ld = seq.selinv(A)
    for k in ("diag", "tip"):
        np.testing.assert_array_equal(L[k], A[k])
        np.testing.assert_array_equal(X[k], A[k])
    assert ld == 0.0


def test_not_positive_definite_reports_global_row():
    A = btagen.g1(5, 5, 4, 2)
    A["diag"][2][1, 1] = -1e6          # row 2*4 + 1 (0-based) -> info 10
    with pytest.raises(seq.NotPositiveDefinite) as ei:
        seq.pobtaf(A)
    assert ei.value.row == 2 * 4 + 1 + 1


def test_not_positive_definite_tip():
    A = btagen.g1(5, 3, 4, 2)
    A["tip"][0, 0] = -1e9
    with pytest.raises(seq.NotPositiveDefinite) as ei:
        seq.pobtaf(A)
    assert ei.value.row == 3 * 4 + 1


def test_trsm_orientations_are_the_ones_that_reproduce_the_inverse():
    # Readings R1/R2: swapping the POBTASI orientation to B L^{-T} breaks the pin.
    A = btagen.g2(2, 5, 4, 2)
    L = seq.pobtaf(A)
    X = seq.pobtasi(L)
    Xd = dense.dense_inverse_pattern(A)
    assert inv.max_block_err(X, Xd)[0] < TOL_X
    saved = seq.trsm_ln
    try:
        seq.trsm_ln = seq.trsm_lt
        Xw = seq.pobtasi(L)
    finally:
        seq.trsm_ln = saved
    assert inv.max_block_err(Xw, Xd)[0] > 1e-3


def test_logdet_fixed_order_deterministic():
    A = btagen.g1(9, 7, 6, 3)
    l1 = seq.selinv(A)[2]
    l2 = seq.selinv(A)[2]
    assert l1 == l2
