"""Pins for oracle/closed_form.py (G2K closed form) and cross-pins of the
oracle recurrences at sizes where the dense expansion is too large -- CPU only."""
import math

import numpy as np
import pytest

import btagen
from oracle import closed_form as cf, dense, invariants as inv, sequential as seq


def test_tridiagonal_inverse_formula():
    # (T^{-1})_{pq} closed form vs numpy.linalg.inv of tridiag(-1, 2+tau, -1)
    for n in (1, 2, 5, 40):
        for tau in (0.1, 1.0):
            T = np.diag(np.full(n, 2 + tau)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)
            Ti = np.linalg.inv(T)
            A, fac = btagen.g2k(1, n, 2, 1, tau=tau, with_factors=True)
            c = cf.closed_form(n, 2, 1, fac)
            for p in range(n):
                for q in range(n):
                    assert abs(c.tinv(p, q) - Ti[p, q]) <= 1e-14 * abs(Ti).max()
            th = c.theta
            ldT = (n + 1) * th + math.log1p(-math.exp(-2 * (n + 1) * th)) - math.log(2 * math.sinh(th))
            assert abs(ldT - np.linalg.slogdet(T)[1]) < 1e-12 * max(1, abs(ldT))


@pytest.mark.parametrize("n,b,a", [(1, 3, 2), (6, 4, 2), (9, 5, 0), (7, 3, 4)])
def test_closed_form_matches_dense_inverse(n, b, a):
    A, fac = btagen.g2k(5, n, b, a, with_factors=True)
    X, ld = cf.selected_inverse(n, b, a, fac)
    e, where = inv.max_block_err(X, dense.dense_inverse_pattern(A))
    assert e < 1e-12, (e, where)
    assert abs(ld - dense.dense_logdet(A)) < 1e-12 * max(1, abs(ld))


def test_oracle_recurrences_match_closed_form_medium():
    # n b = 2048: beyond what the dense pin is used for; the closed form is O(n + b^3)
    n, b, a = 128, 16, 4
    A, fac = btagen.g2k(9, n, b, a, with_factors=True)
    Xc, ldc = cf.selected_inverse(n, b, a, fac)
    L, X, ld = seq.selinv(A)
    e, where = inv.max_block_err(X, Xc)
    assert e < 1e-11, (e, where)
    assert abs(ld - ldc) < 1e-12 * abs(ldc)
    assert inv.llt_residual(L, A) < 1e-13
    assert inv.xa_residual(X, A) < 1e-13
