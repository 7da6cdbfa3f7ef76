"""Plain dense definitions (oracle definition tier; TEST INFRASTRUCTURE ONLY).

PAPER.md Sec. 2.1: a BTA matrix has n diagonal blocks of size b,
lower/upper block diagonals and an arrowhead (last block row/column) whose tip
has size a; N = n b + a.  The factor L keeps the pattern and
POBTASI returns "A^{-1}'s true inverse blocks with the exact same coordinates as
the non-zero blocks of A".  So the plain definitions are: the dense
Cholesky factor of the N x N expansion, and the dense inverse, each restricted
to the BTA pattern.
"""
from __future__ import annotations

import numpy as np


def shapes(A):
    n, b = A["diag"].shape[0], A["diag"].shape[1]
    a = A["tip"].shape[0]
    return n, b, a


def to_dense(A) -> np.ndarray:
    """Place the blocks at their BTA coordinates (arrowhead = last block row/col).

    Symmetric expansion: upper blocks are the transposes of the stored lower
    blocks (A is symmetric, P:302 'symmetric positive-definite').
    """
    n, b, a = shapes(A)
    N = n * b + a
    D = np.zeros((N, N))
    for i in range(n):
        D[i * b:(i + 1) * b, i * b:(i + 1) * b] = A["diag"][i]
        if i + 1 < n:
            D[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = A["lower"][i]
            D[i * b:(i + 1) * b, (i + 1) * b:(i + 2) * b] = A["lower"][i].T
        if a:
            D[n * b:, i * b:(i + 1) * b] = A["arrow"][i]
            D[i * b:(i + 1) * b, n * b:] = A["arrow"][i].T
    if a:
        D[n * b:, n * b:] = A["tip"]
    return D


def to_dense_lower(L) -> np.ndarray:
    """Dense lower-triangular matrix from a BTA factor (no mirroring)."""
    n, b, a = shapes(L)
    N = n * b + a
    D = np.zeros((N, N))
    for i in range(n):
        D[i * b:(i + 1) * b, i * b:(i + 1) * b] = np.tril(L["diag"][i])
        if i + 1 < n:
            D[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b] = L["lower"][i]
        if a:
            D[n * b:, i * b:(i + 1) * b] = L["arrow"][i]
    if a:
        D[n * b:, n * b:] = np.tril(L["tip"])
    return D


def extract_pattern(D: np.ndarray, n: int, b: int, a: int) -> dict:
    """Read back the BTA-pattern blocks (lower half + full diagonal blocks)."""
    out = dict(diag=np.zeros((n, b, b)), lower=np.zeros((max(n - 1, 0), b, b)),
               arrow=np.zeros((n, a, b)), tip=np.zeros((a, a)))
    for i in range(n):
        out["diag"][i] = D[i * b:(i + 1) * b, i * b:(i + 1) * b]
        if i + 1 < n:
            out["lower"][i] = D[(i + 1) * b:(i + 2) * b, i * b:(i + 1) * b]
        if a:
            out["arrow"][i] = D[n * b:, i * b:(i + 1) * b]
    if a:
        out["tip"][:] = D[n * b:, n * b:]
    return out


def dense_cholesky_pattern(A) -> dict:
    """Definition of L: dense Cholesky factor (numpy.linalg) restricted to the pattern."""
    n, b, a = shapes(A)
    return extract_pattern(np.linalg.cholesky(to_dense(A)), n, b, a)


def dense_inverse_pattern(A) -> dict:
    """Definition of X: dense inverse (numpy.linalg.inv) restricted to the pattern."""
    n, b, a = shapes(A)
    return extract_pattern(np.linalg.inv(to_dense(A)), n, b, a)


def dense_logdet(A) -> float:
    sign, ld = np.linalg.slogdet(to_dense(A))
    if sign <= 0:
        raise np.linalg.LinAlgError("matrix is not positive definite")
    return float(ld)
