"""Vendor-library comparator: the paper's own GPU design on B200.

The paper's GPU implementation (§4) calls one cuSOLVER /
cuBLAS routine per block operation from Python (CuPy), with the POBTASI TRSMs
replaced by GEMMs against L_ii^{-1}.  This module is that
design, written with torch.linalg / torch.matmul on a CUDA stream -- i.e.
cusolverDnDpotrf, cublasDtrsm and cublasDgemm calls, one per block operation,
on the same B200 and the same input as our library.  It is a BENCH-ONLY
comparator ("beat the library" bar); it is not part of the product path and
no test or product code calls it.

Block algebra (same orientation readings as DESIGN.md R1-R3):
  POBTAF (Alg. 1)   L_ii = chol(A_ii); L_{i+1,i} = A_{i+1,i} L_ii^{-T};
                                L_{n,i} = A_{n,i} L_ii^{-T}; A_{i+1,i+1} -= L L^T; ...
  POBTASI (Alg. 2)  W_i = L_ii^{-1} (TRSM against I), then GEMM chains.
"""
from __future__ import annotations


def pobtaf(D):
    """In-place blocked Cholesky of the BTA in D (torch CUDA float64); returns log det."""
    import torch
    diag, lower, arrow, tip = D["diag"], D["lower"], D["arrow"], D["tip"]
    n = diag.shape[0]
    a = tip.shape[0]
    logdet = torch.zeros((), dtype=torch.float64, device=diag.device)
    for i in range(n):
        L, _ = torch.linalg.cholesky_ex(diag[i])                          # cusolverDnDpotrf
        diag[i].copy_(L)
        logdet += 2 * torch.log(torch.diagonal(L)).sum()
        LT = L.mT
        if i < n - 1:                                                     # cublasDtrsm (right, lower^T)
            lower[i].copy_(torch.linalg.solve_triangular(LT, lower[i], upper=True, left=False))
            diag[i + 1].addmm_(lower[i], lower[i].mT, alpha=-1.0)         # cublasDgemm (SYRK as GEMM)
        if a:
            arrow[i].copy_(torch.linalg.solve_triangular(LT, arrow[i], upper=True, left=False))
            if i < n - 1:
                arrow[i + 1].addmm_(arrow[i], lower[i].mT, alpha=-1.0)
            tip.addmm_(arrow[i], arrow[i].mT, alpha=-1.0)
    if a:
        Lt, _ = torch.linalg.cholesky_ex(tip)
        tip.copy_(Lt)
        logdet += 2 * torch.log(torch.diagonal(Lt)).sum()
    return logdet


def pobtasi(D):
    """In-place selected inversion from the factor in D (output of pobtaf)."""
    import torch
    diag, lower, arrow, tip = D["diag"], D["lower"], D["arrow"], D["tip"]
    n, b = diag.shape[0], diag.shape[1]
    a = tip.shape[0]
    eye = torch.eye(b, dtype=torch.float64, device=diag.device)
    if a:
        tip.copy_(torch.cholesky_inverse(tip))                            # X_nn = L^{-T} L^{-1}
    Xnn = tip
    for i in range(n - 1, -1, -1):
        W = torch.linalg.solve_triangular(diag[i], eye, upper=False)      # L_ii^{-1} (cublasDtrsm)
        # U terms use the factor blocks of column i before they are overwritten
        if i < n - 1:
            Xlo = -(diag[i + 1] @ lower[i])                               # -X_{i+1,i+1} L_{i+1,i}
            if a:
                Xlo -= arrow[i + 1].mT @ arrow[i]                         # -X_{n,i+1}^T L_{n,i}
            Xlo = Xlo @ W
        if a:
            Xar = -(Xnn @ arrow[i])
            if i < n - 1:
                Xar -= arrow[i + 1] @ lower[i]
            Xar = Xar @ W
        Xd = W.mT.clone()
        if i < n - 1:
            Xd -= Xlo.mT @ lower[i]
        if a:
            Xd -= Xar.mT @ arrow[i]
        diag[i].copy_(Xd @ W)
        if i < n - 1:
            lower[i].copy_(Xlo)
        if a:
            arrow[i].copy_(Xar)
