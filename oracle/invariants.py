"""Size-independent checks (oracle pins; TEST INFRASTRUCTURE ONLY).

  llt_residual   L L^T = A on every pattern block (L is the Cholesky
                 factor and its fill-in stays inside the pattern):
                 (LL^T)_ii     = L_{i,i-1} L_{i,i-1}^T + L_ii L_ii^T
                 (LL^T)_{i+1,i} = L_{i+1,i} L_ii^T
                 (LL^T)_{n,i}   = L_{n,i-1} L_{i,i-1}^T + L_{n,i} L_ii^T
                 (LL^T)_nn     = sum_i L_{n,i} L_{n,i}^T + L_nn L_nn^T
  xa_residual    (X A) = I on the block diagonal, arrow row and tip, using ONLY
                 selected blocks of X (they are the only ones these products touch):
                 (XA)_ii = X_{i,i-1} A_{i-1,i} + X_ii A_ii + X_{i+1,i}^T A_{i+1,i} + X_{n,i}^T A_{n,i}
                 (XA)_{n,i} = X_{n,i-1} A_{i-1,i} + X_{n,i} A_ii + X_{n,i+1} A_{i+1,i} + X_nn A_{n,i}
                 (XA)_nn = sum_i X_{n,i} A_{n,i}^T + X_nn A_nn
  rel_err        relative Frobenius error per block (the parity metric).
"""
from __future__ import annotations

import numpy as np


def rel_err(x: np.ndarray, y: np.ndarray) -> float:
    """||x - y||_F / max(||y||_F, tiny)."""
    d = np.linalg.norm(np.asarray(x) - np.asarray(y))
    r = np.linalg.norm(np.asarray(y))
    if r == 0.0:
        return float(d)
    return float(d / r)


def max_block_err(X, Y, keys=("diag", "lower", "arrow", "tip"), blocks=None):
    """max over blocks of the relative Frobenius error; returns (err, where)."""
    worst, where = 0.0, None
    for k in keys:
        x, y = np.asarray(X[k]), np.asarray(Y[k])
        if k == "tip":
            if y.size:
                e = rel_err(x, y)
                if e > worst:
                    worst, where = e, (k, None)
            continue
        idx = range(y.shape[0]) if blocks is None else [i for i in blocks if i < y.shape[0]]
        for i in idx:
            if y[i].size == 0:
                continue
            e = rel_err(x[i], y[i])
            if e > worst:
                worst, where = e, (k, i)
    return worst, where


def llt_residual(L, A, blocks=None) -> float:
    """max relative residual of L L^T = A over pattern blocks (optionally a subset)."""
    n = A["diag"].shape[0]
    a = A["tip"].shape[0]
    Ld = [np.tril(L["diag"][i]) for i in range(n)]
    worst = 0.0
    idx = range(n) if blocks is None else blocks
    for i in idx:
        R = Ld[i] @ Ld[i].T
        if i > 0:
            R = R + L["lower"][i - 1] @ L["lower"][i - 1].T
        worst = max(worst, rel_err(R, A["diag"][i]))
        if i + 1 < n:
            worst = max(worst, rel_err(L["lower"][i] @ Ld[i].T, A["lower"][i]))
        if a:
            R = L["arrow"][i] @ Ld[i].T
            if i > 0:
                R = R + L["arrow"][i - 1] @ L["lower"][i - 1].T
            worst = max(worst, rel_err(R, A["arrow"][i]))
    if a and blocks is None:
        Lt = np.tril(L["tip"])
        R = Lt @ Lt.T
        for i in range(n):
            R = R + L["arrow"][i] @ L["arrow"][i].T
        worst = max(worst, rel_err(R, A["tip"]))
    return worst


def xa_residual(X, A, blocks=None, scale=None, tip=None) -> float:
    """max abs residual of (XA) - I on diagonal blocks, arrow row and tip,
    normalised by max|A_diag| * max|X_diag| (the scaled residual |XA - I| / (|A| |X|),
    so it is invariant under A -> cA; max over checked blocks).

    blocks: the block rows to check (default all); tip: also check the tip row
    (default: only when all blocks are checked); scale: the normalisation, for
    callers that pass lazily loaded blocks (X[k][i] / A[k][i] are only indexed)."""
    n, b = A["diag"].shape[0], A["diag"].shape[1]
    a = A["tip"].shape[0]
    worst = 0.0
    idx = range(n) if blocks is None else blocks
    if scale is None:
        scale = float(np.abs(A["diag"]).max()) * float(np.abs(X["diag"]).max())
        if not scale > 0.0:
            scale = 1.0
    if tip is None:
        tip = blocks is None
    for i in idx:
        R = X["diag"][i] @ A["diag"][i]
        if i > 0:
            R = R + X["lower"][i - 1] @ A["lower"][i - 1].T
        if i + 1 < n:
            R = R + X["lower"][i].T @ A["lower"][i]
        if a:
            R = R + X["arrow"][i].T @ A["arrow"][i]
        worst = max(worst, float(np.abs(R - np.eye(b)).max()) / scale)
        if a:
            R = X["arrow"][i] @ A["diag"][i] + X["tip"] @ A["arrow"][i]
            if i > 0:
                R = R + X["arrow"][i - 1] @ A["lower"][i - 1].T
            if i + 1 < n:
                R = R + X["arrow"][i + 1] @ A["lower"][i]
            worst = max(worst, float(np.abs(R).max()) / scale)
    if a and tip:
        R = X["tip"] @ A["tip"]
        for i in range(n):
            R = R + X["arrow"][i] @ A["arrow"][i].T
        worst = max(worst, float(np.abs(R - np.eye(a)).max()) / scale)
    return worst
