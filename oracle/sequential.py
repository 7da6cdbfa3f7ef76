"""Block-sequential POBTAF / POBTASI (oracle algorithm tier; TEST INFRASTRUCTURE ONLY).

Follows PAPER.md Alg. 1 (POBTAF) and Alg. 2 (POBTASI)
line by line, on copies of the inputs.  Block primitives are library calls:
POTRF = numpy.linalg.cholesky; TRSM = scipy.linalg.solve_triangular; GEMM = @.

Readings:
  R1 (Alg. 1 l.3-4): TRSM(L_ii, B) = B L_ii^{-T}   (right, lower, transposed).
  R2 (Alg. 2 l.3,5,8,10,12): TRSM(L_ii, U) = U L_ii^{-1} (right, lower, non-transposed).
  R3 (Alg. 2 l.4, l.11): L_ii^{-dagger} is an additive term inside U, then U L_ii^{-1}.
  R4 dagger = transpose (real data).
  R5 log det A = 2 sum log diag(L), summed in the fixed order blocks i ascending,
     entries k ascending, tip last (not in the paper; required by north_star).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


class NotPositiveDefinite(np.linalg.LinAlgError):
    """POTRF met a non-positive pivot.  `row` is the 1-based global row (dpotrf info)."""

    def __init__(self, row: int):
        super().__init__(f"not positive definite: first non-positive pivot at global row {row}")
        self.row = row


def potrf(Aii: np.ndarray, row0: int = 0) -> np.ndarray:
    """L = chol(A), lower.  row0 = global row of A's first row (for the error)."""
    m = Aii.shape[0]
    if m == 0:
        return np.zeros((0, 0))
    try:
        return np.linalg.cholesky(Aii)
    except np.linalg.LinAlgError:
        # locate the first non-positive pivot with the textbook column algorithm
        L = np.tril(np.array(Aii, dtype=np.float64))
        for j in range(m):
            d = L[j, j] - L[j, :j] @ L[j, :j]
            if not d > 0.0:
                raise NotPositiveDefinite(row0 + j + 1) from None
            L[j, j] = np.sqrt(d)
            L[j + 1:, j] = (L[j + 1:, j] - L[j + 1:, :j] @ L[j, :j]) / L[j, j]
        raise  # pragma: no cover


def trsm_lt(L: np.ndarray, B: np.ndarray) -> np.ndarray:
    """Reading R1: X = B L^{-T}, i.e. solve X L^T = B."""
    if B.size == 0:
        return np.array(B, copy=True)
    return sla.solve_triangular(L, B.T, lower=True).T


def trsm_ln(L: np.ndarray, U: np.ndarray) -> np.ndarray:
    """Reading R2: X = U L^{-1}, i.e. solve X L = U."""
    if U.size == 0:
        return np.array(U, copy=True)
    return sla.solve_triangular(L, U.T, lower=True, trans="T").T


def inv_lower(L: np.ndarray) -> np.ndarray:
    """L^{-1} of a lower-triangular block (triangular solve against I)."""
    m = L.shape[0]
    if m == 0:
        return np.zeros((0, 0))
    return sla.solve_triangular(L, np.eye(m), lower=True)


def _copy(A):
    return {k: np.array(A[k], dtype=np.float64, copy=True) for k in ("diag", "lower", "arrow", "tip")}


def logdet_from_factor(L) -> float:
    """R5: 2 * sum log diag over diagonal factors (blocks ascending, entries ascending, tip last)."""
    s = 0.0
    for i in range(L["diag"].shape[0]):
        for v in np.diagonal(L["diag"][i]):
            s += float(np.log(v))
    for v in np.diagonal(L["tip"]):
        s += float(np.log(v))
    return 2.0 * s


def pobtaf(A):
    """POBTAF, Alg. 1.  Returns L (same block layout, strict upper of
    diagonal factors zero).  Raises NotPositiveDefinite with the global pivot row."""
    A = _copy(A)
    n, b = A["diag"].shape[0], A["diag"].shape[1]
    a = A["tip"].shape[0]
    L = _copy(A)
    for i in range(n - 1):                                           # l.1
        L["diag"][i] = potrf(A["diag"][i], i * b)                    # l.2
        L["lower"][i] = trsm_lt(L["diag"][i], A["lower"][i])         # l.3
        L["arrow"][i] = trsm_lt(L["diag"][i], A["arrow"][i])         # l.4
        A["diag"][i + 1] -= L["lower"][i] @ L["lower"][i].T          # l.5
        A["arrow"][i + 1] -= L["arrow"][i] @ L["lower"][i].T         # l.6
        A["tip"] -= L["arrow"][i] @ L["arrow"][i].T                  # l.7
    L["diag"][n - 1] = potrf(A["diag"][n - 1], (n - 1) * b)          # l.9
    L["arrow"][n - 1] = trsm_lt(L["diag"][n - 1], A["arrow"][n - 1])  # l.10
    A["tip"] -= L["arrow"][n - 1] @ L["arrow"][n - 1].T              # l.11
    L["tip"] = potrf(A["tip"], n * b)                                # l.12
    return L


def pobtasi(L):
    """POBTASI, Alg. 2.  Input: factor L from pobtaf.  Returns X with
    X_ii / X_nn full symmetric, X_{i+1,i}, X_{n,i}."""
    L = _copy(L)
    n = L["diag"].shape[0]
    X = _copy(L)
    Wn = inv_lower(L["tip"])
    X["tip"] = Wn.T @ Wn                                                     # l.1
    Ld = L["diag"][n - 1]
    U = -X["tip"] @ L["arrow"][n - 1]                                        # l.2
    X["arrow"][n - 1] = trsm_ln(Ld, U)                                       # l.3
    U = inv_lower(Ld).T - X["arrow"][n - 1].T @ L["arrow"][n - 1]            # l.4
    X["diag"][n - 1] = trsm_ln(Ld, U)                                        # l.5
    for i in range(n - 2, -1, -1):                                           # l.6
        Lii = L["diag"][i]
        U = -X["diag"][i + 1] @ L["lower"][i] - X["arrow"][i + 1].T @ L["arrow"][i]  # l.7
        X["lower"][i] = trsm_ln(Lii, U)                                      # l.8
        U = -X["arrow"][i + 1] @ L["lower"][i] - X["tip"] @ L["arrow"][i]    # l.9
        X["arrow"][i] = trsm_ln(Lii, U)                                      # l.10
        U = (inv_lower(Lii).T - X["lower"][i].T @ L["lower"][i]
             - X["arrow"][i].T @ L["arrow"][i])                              # l.11
        X["diag"][i] = trsm_ln(Lii, U)                                       # l.12
    return X


def selinv(A):
    """POBTAF then POBTASI; returns (L, X, logdet)."""
    L = pobtaf(A)
    X = pobtasi(L)
    return L, X, logdet_from_factor(L)
