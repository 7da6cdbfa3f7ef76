"""Partitioned pipeline PPOBTAF -> POBTARSSI -> PPOBTASI (oracle; TEST INFRASTRUCTURE ONLY).

Follows PAPER.md Sec. 3 in the paper's order:
  plan           Sec. 3.1 partition into P contiguous arrow shapes;
                 top p0 owns A_00, the rest are middle partitions.
  partial_pobtaf Alg. 3 l.3: Alg. 1 lines 1-8 over the top partition,
                 tip updates accumulated in U_0.
  permuted_pobtaf Alg. 4: middle partition with the implicit
                 shifting permutation (first block f = s moved last, never
                 materialised) and the fill-in chain B_i.
  reduced_system Sec. 3.3: the 2P-1 boundary blocks (Fig. 3b-c).
  pobtarssi      POBTAF + POBTASI on A_r.
  partial_pobtasi / permuted_pobtasi  Alg. 5-6, seeded by X_r.

Readings:
  R6  plan: top = floor(r n / (r + P - 1)) clamped to [1, n - 2(P-1)]; the rest
      split evenly over the middles, earlier middles take the remainder.  With
      r = 1 this reproduces Fig. 2's n = 11, P = 3 example whose partition 1
      starts at A_{3,3}.  Minimum sizes: top >= 1, middle >= 2
      (Alg. 4/6 loop bounds P:426, P:484 allow an empty loop).
  R7  B_i is b x b with rows = block f and columns = block i; B_1 = A_{1,0}^T
      (Alg. 4 l.1).
  R8  Alg. 3 l.8 "L_nn <- A_nn + sum U_p" is the pre-factorisation
      reduced tip (U_p are <= 0 downdates); it is factorised in POBTARSSI.
      Sum order: A_nn + U_0 + U_1 + ... (rank ascending).
  R9  Reduced system order [T, F_1, L_1, ..., F_{P-1}, L_{P-1}], T = e_0 - 1,
      F_p = s_p, L_p = e_p - 1; diagonal/arrow blocks = the updated ones;
      lower (F_p, previous) = the ORIGINAL coupling A_{s_p, s_p - 1} (untouched,
      P:389-391); lower (L_p, F_p) = B_{e_p - 1}^T (the final fill-in head).
  R10 "POBTARSSI's result is copied to PPOBTASI's L and B": X_r(L_p,F_p)^T
      seeds the chain Q_{e-1} = X_{f,l}; the output X_{s+1,s} is the final Q_{s+1}^T.
  R11 Alg. 6 typos: l.9 "L^{-dagger} x -X..." drops the spurious "x";
      l.7 "X_{n,0} x L_{0,i}" uses the FACTOR fill-in block B_i (before it is
      overwritten at l.6); l.9 "L_{n,i}" is the partition's arrow block
      L_{n_p,i}; l.10 uses the NEW inverse block Q_i^T times the OLD
      factor B_i, so the factor copy of B_i is kept.
  R12 log det = 2 (sum log diag over the interior factors of all partitions, rank
      ascending, block ascending + all diagonal factors of POBTAF(A_r), tip last).
"""
from __future__ import annotations

import math

import numpy as np

from .sequential import pobtaf, pobtasi, potrf, trsm_lt, trsm_ln, inv_lower, logdet_from_factor


class TooFewBlocks(ValueError):
    pass


def plan(n: int, P: int, r: float = 1.0):
    """Reading R6.  Returns [(s_0, e_0), ..., (s_{P-1}, e_{P-1})]."""
    if P < 1:
        raise TooFewBlocks("P must be >= 1")
    if P == 1:
        if n < 1:
            raise TooFewBlocks("n must be >= 1")
        return [(0, n)]
    if n < 2 * P - 1:
        raise TooFewBlocks(f"n={n} < 2P-1={2 * P - 1}")
    top = int(math.floor(r * n / (r + P - 1)))
    top = max(1, min(top, n - 2 * (P - 1)))
    rest = n - top
    base, rem = divmod(rest, P - 1)
    out = [(0, top)]
    s = top
    for p in range(1, P):
        cnt = base + (1 if (p - 1) < rem else 0)
        out.append((s, s + cnt))
        s += cnt
    assert s == n
    return out


def _copy(A):
    return {k: np.array(A[k], dtype=np.float64, copy=True) for k in ("diag", "lower", "arrow", "tip")}


def partial_pobtaf(W, L, e):
    """Top partition, Alg. 1 lines 1-8 over blocks 0..e-2 (Alg. 3 l.3).
    W: working copy (updated in place); L: factor output.  Returns U_0."""
    a = W["tip"].shape[0]
    b = W["diag"].shape[1]
    U = np.zeros((a, a))
    for i in range(0, e - 1):
        L["diag"][i] = potrf(W["diag"][i], i * b)
        L["lower"][i] = trsm_lt(L["diag"][i], W["lower"][i])
        L["arrow"][i] = trsm_lt(L["diag"][i], W["arrow"][i])
        W["diag"][i + 1] -= L["lower"][i] @ L["lower"][i].T
        W["arrow"][i + 1] -= L["arrow"][i] @ L["lower"][i].T
        U -= L["arrow"][i] @ L["arrow"][i].T
    return U


def permuted_pobtaf(W, L, s, e):
    """Middle partition [s, e), Alg. 4 in global indices (local 0 = f = s).
    Returns (U_p, Bfac, B_last): Bfac[i] = factored fill-in L_{f,i} (R11 keeps it),
    B_last = B_{e-1} (unfactored f-l coupling, rows f, columns l)."""
    a = W["tip"].shape[0]
    b = W["diag"].shape[1]
    f = s
    Bcur = np.array(W["lower"][s].T, copy=True)          # l.1  B_1 = A_{1,0}^T   (R7)
    U = np.zeros((a, a))                                  # l.1  U_tip = 0
    Bfac = {}
    for i in range(s + 1, e - 1):                         # l.2  i = 1 .. n_p - 2
        L["diag"][i] = potrf(W["diag"][i], i * b)         # l.3
        L["lower"][i] = trsm_lt(L["diag"][i], W["lower"][i])   # l.4
        L["arrow"][i] = trsm_lt(L["diag"][i], W["arrow"][i])   # l.5
        Bf = trsm_lt(L["diag"][i], Bcur)                  # l.6
        W["diag"][i + 1] -= L["lower"][i] @ L["lower"][i].T    # l.7
        W["arrow"][i + 1] -= L["arrow"][i] @ L["lower"][i].T   # l.8
        U -= L["arrow"][i] @ L["arrow"][i].T              # l.9
        W["diag"][f] -= Bf @ Bf.T                         # l.10
        Bcur = -Bf @ L["lower"][i].T                      # l.11
        W["arrow"][f] -= L["arrow"][i] @ Bf.T             # l.12
        Bfac[i] = Bf
    return U, Bfac, Bcur


def reduced_system(W, A, parts, Us, Blast):
    """Reading R9: assemble A_r with n_r = 2P - 1 diagonal blocks (Sec. 3.3)."""
    P = len(parts)
    b = W["diag"].shape[1]
    a = W["tip"].shape[0]
    nr = 2 * P - 1
    Ar = dict(diag=np.zeros((nr, b, b)), lower=np.zeros((nr - 1, b, b)),
              arrow=np.zeros((nr, a, b)), tip=np.array(A["tip"], copy=True))
    T = parts[0][1] - 1
    Ar["diag"][0] = W["diag"][T]
    Ar["arrow"][0] = W["arrow"][T]
    for p in range(1, P):
        s, e = parts[p]
        Ar["diag"][2 * p - 1] = W["diag"][s]
        Ar["arrow"][2 * p - 1] = W["arrow"][s]
        Ar["diag"][2 * p] = W["diag"][e - 1]
        Ar["arrow"][2 * p] = W["arrow"][e - 1]
        Ar["lower"][2 * p - 2] = A["lower"][s - 1]        # original coupling (F_p, previous)
        Ar["lower"][2 * p - 1] = Blast[p].T               # (L_p, F_p) = B_{e-1}^T
    for p in range(P):                                     # R8: rank-ascending sum
        Ar["tip"] = Ar["tip"] + Us[p]
    return Ar


def pobtarssi(Ar):
    """POBTARSSI (Sec. 3.3): block-sequential POBTAF + POBTASI on A_r."""
    Lr = pobtaf(Ar)
    Xr = pobtasi(Lr)
    return Lr, Xr


def partial_pobtasi(L, X, e, Xr, P):
    """Top partition: Alg. 2 lines 6-13 for i = e-2 .. 0 seeded by X_r."""
    T = e - 1
    X["diag"][T] = Xr["diag"][0]
    X["arrow"][T] = Xr["arrow"][0]
    if P > 1:
        X["lower"][T] = Xr["lower"][0]
    for i in range(e - 2, -1, -1):
        Lii = L["diag"][i]
        U = -X["diag"][i + 1] @ L["lower"][i] - X["arrow"][i + 1].T @ L["arrow"][i]
        X["lower"][i] = trsm_ln(Lii, U)
        U = -X["arrow"][i + 1] @ L["lower"][i] - X["tip"] @ L["arrow"][i]
        X["arrow"][i] = trsm_ln(Lii, U)
        U = inv_lower(Lii).T - X["lower"][i].T @ L["lower"][i] - X["arrow"][i].T @ L["arrow"][i]
        X["diag"][i] = trsm_ln(Lii, U)


def permuted_pobtasi(L, X, s, e, Bfac, Xr, p, P):
    """Middle partition [s, e): Alg. 6 with readings R10, R11."""
    f, l = s, e - 1
    X["diag"][f] = Xr["diag"][2 * p - 1]
    X["arrow"][f] = Xr["arrow"][2 * p - 1]
    X["diag"][l] = Xr["diag"][2 * p]
    X["arrow"][l] = Xr["arrow"][2 * p]
    if p < P - 1:
        X["lower"][l] = Xr["lower"][2 * p]                 # (F_{p+1}, L_p)
    Q = np.array(Xr["lower"][2 * p - 1].T, copy=True)      # Q_{e-1} = X_{f,l}   (R10)
    Xff, Xnf, Xnn = X["diag"][f], X["arrow"][f], X["tip"]
    for i in range(e - 2, s, -1):                          # l.1  i = n_p-2 .. 1
        Lii = L["diag"][i]
        Lf = Bfac[i]                                       # factor L_{f,i} (R11)
        U = -X["diag"][i + 1] @ L["lower"][i] - X["arrow"][i + 1].T @ L["arrow"][i]   # l.2
        U = U - Q.T @ Lf                                                              # l.3
        X["lower"][i] = trsm_ln(Lii, U)                                               # l.4
        V = -Q @ L["lower"][i] - Xff @ Lf - Xnf.T @ L["arrow"][i]                     # l.5
        Qn = trsm_ln(Lii, V)                                                          # l.6
        U = -X["arrow"][i + 1] @ L["lower"][i] - Xnn @ L["arrow"][i]                  # l.7
        U = U - Xnf @ Lf                                                              # l.8
        X["arrow"][i] = trsm_ln(Lii, U)                                               # l.9
        U = inv_lower(Lii).T - X["lower"][i].T @ L["lower"][i] - X["arrow"][i].T @ L["arrow"][i]  # l.10
        U = U - Qn.T @ Lf                                                             # l.11
        X["diag"][i] = trsm_ln(Lii, U)                                                # l.12
        Q = Qn
    X["lower"][s] = Q.T                                    # X_{s+1,s} = Q_{s+1}^T   (R10)


def _logdiag(M):
    s = 0.0
    for v in np.diagonal(M):
        s += float(np.log(v))
    return s


def pselinv(A, P: int, r: float = 1.0):
    """In-process P-partition pipeline (Fig. 3).  Returns a dict with
    L (eliminated factor blocks; boundary blocks hold their updated values W),
    W (working matrix after PPOBTAF), X, logdet, parts, Ar, Lr, Xr, Bfac, Blast, U."""
    A = _copy(A)
    n = A["diag"].shape[0]
    parts = plan(n, P, r)
    W = _copy(A)
    L = _copy(A)
    Us, Bfacs, Blast = [None] * P, [None] * P, [None] * P
    # PPOBTAF (Alg. 3): partitions are independent
    Us[0] = partial_pobtaf(W, L, parts[0][1])
    for p in range(1, P):
        s, e = parts[p]
        Us[p], Bfacs[p], Blast[p] = permuted_pobtaf(W, L, s, e)
    # boundary blocks of L hold the updated (not yet factorised) values
    bnd = [parts[0][1] - 1] + [x for p in range(1, P) for x in (parts[p][0], parts[p][1] - 1)]
    for k in bnd:
        L["diag"][k] = W["diag"][k]
        L["arrow"][k] = W["arrow"][k]
    # POBTARSSI
    Ar = reduced_system(W, A, parts, Us, Blast)
    Lr, Xr = pobtarssi(Ar)
    # PPOBTASI (Alg. 5)
    X = _copy(A)
    X["tip"] = np.array(Xr["tip"], copy=True)
    partial_pobtasi(L, X, parts[0][1], Xr, P)
    for p in range(1, P):
        s, e = parts[p]
        permuted_pobtasi(L, X, s, e, Bfacs[p], Xr, p, P)
    # log det (R12)
    ld = 0.0
    for i in range(0, parts[0][1] - 1):
        ld += _logdiag(L["diag"][i])
    for p in range(1, P):
        s, e = parts[p]
        for i in range(s + 1, e - 1):
            ld += _logdiag(L["diag"][i])
    ld = 2.0 * ld + logdet_from_factor(Lr)
    return dict(L=L, W=W, X=X, logdet=ld, parts=parts, Ar=Ar, Lr=Lr, Xr=Xr,
                Bfac=Bfacs, Blast=Blast, U=Us)
