"""Seeded synthetic SPD BTA input generators (shared by tests, the oracle's callers and bench).

This module holds NO arithmetic of the method (no factorization, no inversion):
it only produces input matrices with the BTA structure of PAPER.md §2.1
(Table 2: n diagonal blocks of size b, lower blocks A_{i+1,i},
arrow blocks A_{n,i} of size a x b, tip A_{n,n} of size a x a, N = nb + a).
It is imported by tests/ and bench.py; neither oracle/ nor the CUDA product path
imports it, so it is the one module both sides of a parity test share.

Storage convention (the C-ABI layout, include/serinv.h): four C-contiguous
float64 arrays
    diag  [n][b][b]    A_{i,i}     (full symmetric blocks)
    lower [n-1][b][b]  A_{i+1,i}
    arrow [n][a][b]    A_{n,i}
    tip   [a][a]       A_{n,n}     (full symmetric)

Generators (recipes):

G1 "diagonally dominant"  (BASELINE north_star: "seeded, diagonally dominated
    SPD generators"; the synthetic dataset (1) of P:688 gives shapes only).
    Every off-diagonal entry of the pattern is u(i,j) = k * 2^-23 - 1 with
    k = splitmix64(seed, stream, min(i,j), max(i,j)) >> 40 (24 random bits), so
    u in [-1, 1) is symmetric in (i,j) and exactly representable.  Each
    diagonal entry is set to 1 + sum_{j != i, j in pattern row} |u(i,j)|.
    Because every |u| is a multiple of 2^-23 and the row sums stay below
    2^29, the sum is EXACT in float64 in any order, so any producer of this
    recipe (host or device) gives bit-identical values.  SPD by Gershgorin.

G2 "Kronecker / SPDE-like" (the paper's spatio-temporal structure):
    A_ii = (2 + tau) M + eps S_i,  A_{i+1,i} = -M,  eps = tau / (2b),
    M = a G1-style SPD b x b block (lambda_min(M) >= 1 by Gershgorin),
    S_i symmetric with entries u in [-1, 1)  (||eps S_i||_2 <= tau/2),
    arrow W_i entries u / sqrt(n b)  (||W||_F^2 <= a),
    tip = (1 + 2a/tau) I + symmetric noise with row sums < 1/2.
    SPD: lambda_min(T (x) M + eps S) >= tau/2, and the tip's Schur complement
    is >= 1 + 2a/tau - 1/2 - a / (tau/2) = 1/2.  Fill-in decays ~0.73 per block
    (root of x^2 - (2+tau) x + 1), so errors deep inside middle partitions stay
    visible (unlike G1 where the fill-in decays ~1/sqrt(b) per block).

G2K = G2 with eps = 0 and W_i = w_i V (a x b), the case with a closed-form
    selected inverse (oracle/closed_form.py).  `g2k` also returns the factors
    (M, V, w, C, tau) so the closed form can be evaluated.
"""
from __future__ import annotations

import numpy as np

__all__ = ["g1", "g2", "g2k", "generate", "bta_bytes", "BTA"]

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_SCALE = 2.0 ** -23

# stream ids (distinct hash domains)
S_G1, S_M, S_S, S_W, S_TIPN, S_V, S_w = 1, 2, 3, 4, 5, 6, 7


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def _seedkey(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _GOLD + np.uint64(stream) * _M2
        return _mix(np.asarray(s + _GOLD, dtype=np.uint64))[()]


def _u(seed: int, stream: int, i, j):
    """Symmetric hash-uniform u(i,j) in [-1,1), multiple of 2^-23 (exact)."""
    i = np.asarray(i, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    lo = np.minimum(i, j)
    hi = np.maximum(i, j)
    with np.errstate(over="ignore"):
        key = ((hi << np.uint64(32)) | lo) ^ _seedkey(seed, stream)
        h = _mix(key + _GOLD)
    return (h >> np.uint64(40)).astype(np.float64) * _SCALE - 1.0


def _u_block(seed, stream, r0, c0, nr, nc):
    r = np.arange(r0, r0 + nr, dtype=np.uint64)[:, None]
    c = np.arange(c0, c0 + nc, dtype=np.uint64)[None, :]
    return _u(seed, stream, r, c)


class BTA(dict):
    """dict with keys diag, lower, arrow, tip (+ n, b, a attributes)."""

    @property
    def n(self):
        return self["diag"].shape[0]

    @property
    def b(self):
        return self["diag"].shape[1]

    @property
    def a(self):
        return self["tip"].shape[0]

    def copy(self):
        out = BTA({k: np.array(v, copy=True) for k, v in self.items() if isinstance(v, np.ndarray)})
        for k, v in self.items():
            if not isinstance(v, np.ndarray):
                out[k] = v
        return out


def bta_bytes(n: int, b: int, a: int) -> int:
    return 8 * (n * b * b + max(n - 1, 0) * b * b + n * a * b + a * a)


def _alloc(n, b, a):
    return BTA(diag=np.zeros((n, b, b)), lower=np.zeros((max(n - 1, 0), b, b)),
               arrow=np.zeros((n, a, b)), tip=np.zeros((a, a)))


def g1(seed: int, n: int, b: int, a: int) -> BTA:
    """G1: diagonally dominant dense-block SPD BTA (recipe in the module doc)."""
    A = _alloc(n, b, a)
    N0 = n * b  # first tip row (global)
    rowsum = np.zeros(n * b)
    tipsum = np.zeros(a)
    for i in range(n):
        D = _u_block(seed, S_G1, i * b, i * b, b, b)
        np.fill_diagonal(D, 0.0)
        A["diag"][i] = D
        rowsum[i * b:(i + 1) * b] += np.abs(D).sum(axis=1)
        if i + 1 < n:
            Lw = _u_block(seed, S_G1, (i + 1) * b, i * b, b, b)
            A["lower"][i] = Lw
            rowsum[(i + 1) * b:(i + 2) * b] += np.abs(Lw).sum(axis=1)
            rowsum[i * b:(i + 1) * b] += np.abs(Lw).sum(axis=0)
        if a:
            W = _u_block(seed, S_G1, N0, i * b, a, b)
            A["arrow"][i] = W
            rowsum[i * b:(i + 1) * b] += np.abs(W).sum(axis=0)
            tipsum += np.abs(W).sum(axis=1)
    for i in range(n):
        idx = np.arange(b)
        A["diag"][i][idx, idx] = 1.0 + rowsum[i * b:(i + 1) * b]
    if a:
        Tt = _u_block(seed, S_G1, N0, N0, a, a)
        np.fill_diagonal(Tt, 0.0)
        tipsum += np.abs(Tt).sum(axis=1)
        Tt[np.arange(a), np.arange(a)] = 1.0 + tipsum
        A["tip"][:] = Tt
    A["gen"] = ("g1", seed)
    return A


def _spd_M(seed: int, b: int) -> np.ndarray:
    M = _u_block(seed, S_M, 0, 0, b, b)
    np.fill_diagonal(M, 0.0)
    s = np.abs(M).sum(axis=1)
    M[np.arange(b), np.arange(b)] = 1.0 + s
    return M


def _tip_noise(seed: int, a: int, tau: float) -> np.ndarray:
    C = _u_block(seed, S_TIPN, 0, 0, a, a) * (0.5 / max(a, 1))
    np.fill_diagonal(C, 0.0)
    C[np.arange(a), np.arange(a)] = 1.0 + 2.0 * a / tau
    return C


def g2(seed: int, n: int, b: int, a: int, tau: float = 0.1) -> BTA:
    """G2: Kronecker / SPDE-like SPD BTA (recipe in the module doc)."""
    A = _alloc(n, b, a)
    M = _spd_M(seed, b)
    eps = tau / (2.0 * b)
    c = 2.0 + tau
    for i in range(n):
        S = _u_block(seed, S_S, i * b, i * b, b, b)
        A["diag"][i] = c * M + eps * S
        if i + 1 < n:
            A["lower"][i] = -M
        if a:
            A["arrow"][i] = _u_block(seed, S_W, n * b, i * b, a, b) * (1.0 / np.sqrt(n * b))
    if a:
        A["tip"][:] = _tip_noise(seed, a, tau)
    A["gen"] = ("g2", seed)
    return A


def g2k(seed: int, n: int, b: int, a: int, tau: float = 0.1, with_factors: bool = False):
    """G2K: G2 with eps = 0 and W_i = w_i V (closed-form selected inverse).

    Returns the BTA, and with with_factors=True also dict(M, V, w, C, tau).
    """
    A = _alloc(n, b, a)
    M = _spd_M(seed, b)
    c = 2.0 + tau
    D = c * M
    V = _u_block(seed, S_V, 0, 0, a, b) * (1.0 / np.sqrt(b)) if a else np.zeros((0, b))
    w = _u_block(seed, S_w, 0, 0, 1, n)[0] * (1.0 / np.sqrt(n))
    for i in range(n):
        A["diag"][i] = D
        if i + 1 < n:
            A["lower"][i] = -M
        if a:
            A["arrow"][i] = w[i] * V
    C = _tip_noise(seed, a, tau) if a else np.zeros((0, 0))
    A["tip"][:] = C
    A["gen"] = ("g2k", seed)
    if with_factors:
        return A, dict(M=M, V=V, w=w, C=C, tau=tau)
    return A


def generate(kind: str, seed: int, n: int, b: int, a: int, **kw) -> BTA:
    kind = kind.lower()
    if kind == "g1":
        return g1(seed, n, b, a)
    if kind == "g2":
        return g2(seed, n, b, a, **kw)
    if kind == "g2k":
        return g2k(seed, n, b, a, **kw)
    raise ValueError(f"unknown generator {kind!r}")


# --------------------------------------------------------------------------- device twin
# The same counter-based recipe in torch int64 arithmetic (wrapping multiply,
# logical shifts by masking), so large inputs can be generated directly in HBM.
# Bit-identical to the numpy path (tests/test_generators.py checks it on CPU).
def _t_consts():
    def s64(x):
        x &= 0xFFFFFFFFFFFFFFFF
        return x - (1 << 64) if x >= (1 << 63) else x
    return s64(0x9E3779B97F4A7C15), s64(0xBF58476D1CE4E5B9), s64(0x94D049BB133111EB)


def _t_shr(x, k):
    return (x >> k) & ((1 << (64 - k)) - 1)


def _t_mix(z):
    _, m1, m2 = _t_consts()
    z = (z ^ _t_shr(z, 30)) * m1
    z = (z ^ _t_shr(z, 27)) * m2
    return z ^ _t_shr(z, 31)


def _t_seedkey(seed, stream):
    import torch
    gold, _, m2 = _t_consts()
    s = torch.tensor([seed & 0x7FFFFFFFFFFFFFFF], dtype=torch.int64)
    s = s * gold + stream * m2
    return int(_t_mix(s + gold)[0])


def _t_u_block(seed, stream, r0, c0, nr, nc, device):
    import torch
    gold, _, _ = _t_consts()
    r = torch.arange(r0, r0 + nr, dtype=torch.int64, device=device)[:, None]
    c = torch.arange(c0, c0 + nc, dtype=torch.int64, device=device)[None, :]
    lo = torch.minimum(r, c)
    hi = torch.maximum(r, c)
    key = ((hi << 32) | lo) ^ _t_seedkey(seed, stream)
    h = _t_mix(key + gold)
    return _t_shr(h, 40).to(torch.float64) * _SCALE - 1.0


def g1_torch(seed: int, n: int, b: int, a: int, device="cuda", start: int = 0, end: int | None = None):
    """G1 generated with torch on `device` (dict of tensors, C-ABI layout);
    bit-identical to g1(seed, n, b, a).  With a block range [start, end) it
    returns the rank-local slice used by the distributed path: diag/arrow
    [end-start], lower [end-start] (the coupling to the next rank included) or
    [end-start-1] on the last rank, and the (replicated) tip.  Seeds < 2^63."""
    import torch
    end = n if end is None else end
    cnt = end - start
    last = end == n
    nl = cnt - 1 if last else cnt
    out = {"diag": torch.empty((cnt, b, b), dtype=torch.float64, device=device),
           "lower": torch.empty((max(nl, 0), b, b), dtype=torch.float64, device=device),
           "arrow": torch.empty((cnt, a, b), dtype=torch.float64, device=device),
           "tip": torch.empty((a, a), dtype=torch.float64, device=device)}
    N0 = n * b
    rowsum = torch.zeros(cnt * b, dtype=torch.float64, device=device)
    eye = torch.eye(b, dtype=torch.bool, device=device)
    for i in range(max(0, start - 1), end):
        if i >= start:
            D = _t_u_block(seed, S_G1, i * b, i * b, b, b, device)
            D.masked_fill_(eye, 0.0)
            out["diag"][i - start] = D
            rowsum[(i - start) * b:(i - start + 1) * b] += D.abs().sum(dim=1)
        if i + 1 < n:
            Lw = _t_u_block(seed, S_G1, (i + 1) * b, i * b, b, b, device)
            if i >= start and i - start < nl:
                out["lower"][i - start] = Lw
            if start <= i + 1 < end:
                rowsum[(i + 1 - start) * b:(i + 2 - start) * b] += Lw.abs().sum(dim=1)
            if i >= start:
                rowsum[(i - start) * b:(i - start + 1) * b] += Lw.abs().sum(dim=0)
    tipsum = torch.zeros(a, dtype=torch.float64, device=device)
    if a:
        for i in range(n):  # the tip's diagonal needs every arrow block
            W = _t_u_block(seed, S_G1, N0, i * b, a, b, device)
            if start <= i < end:
                out["arrow"][i - start] = W
                rowsum[(i - start) * b:(i - start + 1) * b] += W.abs().sum(dim=0)
            tipsum += W.abs().sum(dim=1)
    idx = torch.arange(b, device=device)
    for i in range(cnt):
        out["diag"][i][idx, idx] = 1.0 + rowsum[i * b:(i + 1) * b]
    if a:
        Tt = _t_u_block(seed, S_G1, N0, N0, a, a, device)
        Tt.masked_fill_(torch.eye(a, dtype=torch.bool, device=device), 0.0)
        tipsum += Tt.abs().sum(dim=1)
        ia = torch.arange(a, device=device)
        Tt[ia, ia] = 1.0 + tipsum
        out["tip"].copy_(Tt)
    return out
