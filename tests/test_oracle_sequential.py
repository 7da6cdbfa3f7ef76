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


# ---------------------------------------------------------------------------
# Sensitivity pins of the size-independent checkers.  The -m gpu
# full-size tests at C3 use xa_residual on sampled blocks as their parity
# property, so it must fail on small errors:
#   xa_residual (scaled |XA - I| / (max|A| max|X|)): exact results give < 1e-13; an
#     error of 1e-8 * max|X_diag| in ONE entry of any selected block gives >= 1e-9
#     (it bounds absolute errors relative to the largest entry of X);
#   llt_residual (relative Frobenius per pattern block): an error of 1e-8 ||L_blk||_F
#     in one entry gives >= 1e-9.

@pytest.mark.parametrize("key,blk", [("diag", 0), ("diag", 3), ("arrow", 0), ("arrow", 7), ("tip", None)])
@pytest.mark.parametrize("gen", ["g1", "g2"])
def test_xa_residual_detects_a_1e8_perturbation(key, blk, gen):
    A = btagen.generate(gen, 3, 8, 16, 3)
    L, X, ld = seq.selinv(A)
    assert inv.xa_residual(X, A) < 1e-13
    for r, c in ((1, 2), (2, 2), (0, 15 if key != "tip" else 2)):
        Xp = {k: v.copy() for k, v in X.items()}
        T = Xp[key] if blk is None else Xp[key][blk]
        T[r, c] += 1e-8 * np.abs(X["diag"]).max()
        if key in ("diag", "tip"):   # X_ii / X_nn are stored full symmetric
            T[c, r] = T[r, c]
        res = inv.xa_residual(Xp, A)
        assert res >= 1e-9, (r, c, res)
        # the sampled form the GPU tests use sees it too when the block's row is sampled
        assert (inv.xa_residual(Xp, A, blocks=[0, 7], tip=True) if key == "tip"
                else inv.xa_residual(Xp, A, blocks=[blk])) >= 1e-9


@pytest.mark.parametrize("gen", ["g1", "g2"])
@pytest.mark.parametrize("mutation", ["lower_sign", "lower_transposed", "lower_zero", "lower_shifted",
                                      "arrow_sign", "diag_swapped", "tip_dropped_term"])
def test_xa_residual_detects_plausible_mistakes(gen, mutation):
    # X_{i+1,i} enters (XA)|pattern only through products with the off-diagonal
    # blocks of A, so a 1e-8 error in it is scaled by |A_{i+1,i}| / |A_ii| there;
    # the mistakes a wrong implementation makes (sign, transposed operand, dropped
    # or misplaced block) change it by O(|X_{i+1,i}|) and are caught by far.
    A = btagen.generate(gen, 6, 8, 16, 3)
    L, X, ld = seq.selinv(A)
    Xp = {k: v.copy() for k, v in X.items()}
    i = 3
    if mutation == "lower_sign":
        Xp["lower"][i] = -Xp["lower"][i]
    elif mutation == "lower_transposed":
        Xp["lower"][i] = Xp["lower"][i].T.copy()
    elif mutation == "lower_zero":
        Xp["lower"][i] = 0.0
    elif mutation == "lower_shifted":
        Xp["lower"][i] = X["lower"][i + 1]
    elif mutation == "arrow_sign":
        Xp["arrow"][i] = -Xp["arrow"][i]
    elif mutation == "diag_swapped":
        Xp["diag"][i] = X["diag"][i + 1]
    else:   # tip without the arrow contributions' final term
        Xp["tip"] = np.linalg.inv(A["tip"])
    assert inv.xa_residual(Xp, A, blocks=[i, i + 1], tip=True) >= 1e-9


@pytest.mark.parametrize("key,blk", [("diag", 0), ("diag", 5), ("lower", 3), ("arrow", 7), ("tip", None)])
def test_llt_residual_detects_a_1e8_perturbation(key, blk):
    A = btagen.g1(4, 8, 16, 3)
    L, X, ld = seq.selinv(A)
    assert inv.llt_residual(L, A) < 1e-13
    Lp = {k: v.copy() for k, v in L.items()}
    T = Lp[key] if blk is None else Lp[key][blk]
    T[2, 1] += 1e-8 * np.linalg.norm(T)
    assert inv.llt_residual(Lp, A) >= 1e-9


def test_xa_residual_lazy_blocks_and_scale():
    # the GPU tests pass lazily fetched blocks and an explicit scale: same value
    A = btagen.g2(2, 9, 12, 2)
    L, X, ld = seq.selinv(A)

    class Lazy:
        def __init__(self, arr):
            self.arr = arr
            self.shape = arr.shape

        def __getitem__(self, i):
            return self.arr[i]
    scale = float(np.abs(A["diag"]).max()) * float(np.abs(X["diag"]).max())
    keys = ("diag", "lower", "arrow")
    XL = {k: Lazy(X[k]) for k in keys} | {"tip": X["tip"]}
    AL = {k: Lazy(A[k]) for k in keys} | {"tip": A["tip"]}
    blocks = [0, 4, 8]
    assert inv.xa_residual(XL, AL, blocks=blocks, scale=scale, tip=True) == \
        inv.xa_residual(X, A, blocks=blocks, tip=True)
