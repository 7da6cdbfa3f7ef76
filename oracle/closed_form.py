"""Closed-form selected inverse of the G2K Kronecker BTA (oracle pin; TEST INFRASTRUCTURE ONLY).

A = [[T (x) M, W^T], [W, C]] with T = tridiag(-1, d, -1) (n x n), d = 2 + tau,
M SPD (b x b), W = w^T (x) V (block i = w_i V, a x b), C SPD (a x a).
Block-matrix inversion (Schur complement on the tip) gives, with
K = T (x) M, K^{-1} = T^{-1} (x) M^{-1}, t = T^{-1} w, G = V M^{-1} V^T:

  S      = C - (w^T t) G                       (Schur complement of the tip)
  X_nn   = S^{-1}
  X_{n,p} = -t_p S^{-1} V M^{-1}
  X_{pq} = (T^{-1})_{pq} M^{-1} + t_p t_q Z,   Z = M^{-1} V^T S^{-1} V M^{-1}
  log det A = b log det T + n log det M + log det S

and, with d = 2 cosh(theta), for p <= q (0-based; overflow-free form)
  (T^{-1})_{pq} = e^{-(q-p) theta} (1 - e^{-2(p+1) theta}) (1 - e^{-2(n-q) theta})
                  / (2 sinh(theta) (1 - e^{-2(n+1) theta}))
  log det T = (n+1) theta + log1p(-e^{-2(n+1) theta}) - log(2 sinh theta).

This is the plain definition of A^{-1} on the BTA pattern for this family
(P:357); it shares no step with the block recurrences of Alg. 1-2.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla


class G2KClosedForm:
    def __init__(self, n, b, a, M, V, w, C, tau):
        self.n, self.b, self.a = n, b, a
        self.theta = math.acosh(1.0 + tau / 2.0)           # d = 2 + tau = 2 cosh(theta)
        self.Minv = np.linalg.inv(M)
        self.Minv = 0.5 * (self.Minv + self.Minv.T)
        # t = T^{-1} w  (banded solve of the tridiagonal T)
        d = 2.0 + tau
        ab = np.zeros((3, n))
        ab[0, 1:] = -1.0
        ab[1, :] = d
        ab[2, :-1] = -1.0
        self.t = sla.solve_banded((1, 1), ab, np.asarray(w, dtype=np.float64))
        self.w = np.asarray(w, dtype=np.float64)
        if a:
            VM = V @ self.Minv                              # a x b
            G = VM @ V.T
            S = C - float(self.w @ self.t) * G
            self.Sinv = np.linalg.inv(S)
            self.Sinv = 0.5 * (self.Sinv + self.Sinv.T)
            self.SVM = self.Sinv @ VM                       # S^{-1} V M^{-1}
            self.Z = VM.T @ self.SVM                        # M^{-1} V^T S^{-1} V M^{-1}
            sgn, ldS = np.linalg.slogdet(S)
            assert sgn > 0
            self.ldS = ldS
        else:
            self.Sinv = np.zeros((0, 0))
            self.SVM = np.zeros((0, b))
            self.Z = np.zeros((b, b))
            self.ldS = 0.0
        sgn, ldM = np.linalg.slogdet(M)
        assert sgn > 0
        self.ldM = ldM

    def tinv(self, p: int, q: int) -> float:
        if p > q:
            p, q = q, p
        th, n = self.theta, self.n
        num = math.exp(-(q - p) * th) * (-math.expm1(-2 * (p + 1) * th)) * (-math.expm1(-2 * (n - q) * th))
        den = 2.0 * math.sinh(th) * (-math.expm1(-2 * (n + 1) * th))
        return num / den

    def X_block(self, p: int, q: int) -> np.ndarray:
        """X_{pq} (b x b) for any p, q (the pattern uses |p - q| <= 1)."""
        return self.tinv(p, q) * self.Minv + self.t[p] * self.t[q] * self.Z

    def X_arrow(self, p: int) -> np.ndarray:
        return -self.t[p] * self.SVM

    def X_tip(self) -> np.ndarray:
        return self.Sinv

    def logdet(self) -> float:
        th, n = self.theta, self.n
        ldT = (n + 1) * th + math.log1p(-math.exp(-2 * (n + 1) * th)) - math.log(2 * math.sinh(th))
        return self.b * ldT + n * self.ldM + self.ldS


def closed_form(n, b, a, factors) -> G2KClosedForm:
    f = factors
    return G2KClosedForm(n, b, a, f["M"], f["V"], f["w"], f["C"], f["tau"])


def selected_inverse(n, b, a, factors) -> dict:
    """Full pattern of X from the closed form (cost O(n b^2) to materialise)."""
    cf = closed_form(n, b, a, factors)
    X = dict(diag=np.zeros((n, b, b)), lower=np.zeros((max(n - 1, 0), b, b)),
             arrow=np.zeros((n, a, b)), tip=np.array(cf.X_tip(), copy=True))
    for i in range(n):
        X["diag"][i] = cf.X_block(i, i)
        if i + 1 < n:
            X["lower"][i] = cf.X_block(i + 1, i)
        if a:
            X["arrow"][i] = cf.X_arrow(i)
    return X, cf.logdet()
