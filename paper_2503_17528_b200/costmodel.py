"""Analytic cost model of the partitioned method: load balancing and parallel
efficiency (Sec. 4.3 "Load balancing" P:608-614, Table 4 P:595-606,
Sec. 4.4 "Parallel efficiency" P:627-633, Fig. 3a).

Host-side arithmetic on flop counts only (no matrix data); it plans, it does not
compute the method.  Flops use LAPACK leading-order counting (SURVEY 8(a):
POTRF m^3/3, TRSM/TRMM r m^2, SYRK m^2 k, GEMM 2mnk), per eliminated block:

  top / bottom partition (no fill-in; Alg. 1 + Alg. 2 rows a1-a12)
    F_end = 7/3 b^3 + 3 a b^2 + a^2 b            S_end = 14/3 b^3 + 6 a b^2 + 2 a^2 b
  middle partition (Alg. 4 fill-in chain B_i, Alg. 6 chain Q_i = X_{f,i})
    F_mid = F_end + 4 b^3 + 2 a b^2              (TRSM of B_i, A_ff -= L_fi L_fi^T,
                                                  B_{i+1} = -L_fi L_{i+1,i}^T, A_nf -= L_ni L_fi^T)
    S_mid = S_end + 8 b^3 + 4 a b^2              (L_fi W_i, Q_i = -Q_{i+1} L'_i - X_ff L'_fi
                                                  - X_nf^T L'n_i, -Q_{i+1}^T L'_fi, -X_nf L'_fi,
                                                  -Q_i^T L'_fi)
  reduced system: POBTAF + POBTASI of its blocks (block-sequential POBTARSSI).

A partition of k blocks eliminates k - 1 (top / bottom: its boundary block joins
the reduced system) or k - 2 (middle: first and last block) of them (Table 3's
n/P - 2).

Load balancing (Sec. 4.3): r = n_top / n_mid such that the top and a middle
partition do the same work, separately for the factorisation (r_F) and the
inversion (r_S); Table 4 combines them with the PPOBTAF / PPOBTASI operation
ratio rho.  Reading: r_LB = rho r_F + (1 - rho) r_S.

Parallel efficiency (Sec. 4.4): E(n, P) = W_seq(n) / (P W_proc(n, P)) with
W_proc = the busiest partition's work + the reduced system's work (the
block-sequential POBTARSSI every process waits for).

`scheme="paper"`: P - 1 middle partitions, 2P - 1 reduced blocks (Sec. 3).
`scheme="twisted"`: the last partition eliminates bottom-up without fill-in
(reading R14): P - 2 middle partitions, 2P - 2 reduced blocks, both
end partitions r times a middle one.
"""
from __future__ import annotations

from dataclasses import dataclass


def f_end(b: float, a: float) -> float:
    return 7 / 3 * b ** 3 + 3 * a * b * b + a * a * b


def s_end(b: float, a: float) -> float:
    return 14 / 3 * b ** 3 + 6 * a * b * b + 2 * a * a * b


def f_mid(b: float, a: float) -> float:
    return f_end(b, a) + 4 * b ** 3 + 2 * a * b * b


def s_mid(b: float, a: float) -> float:
    return s_end(b, a) + 8 * b ** 3 + 4 * a * b * b


def f_seq(n: int, b: float, a: float) -> float:
    """POBTAF of n blocks."""
    return (n - 1) * f_end(b, a) + b ** 3 / 3 + a * b * b + a * a * b + a ** 3 / 3


def s_seq(n: int, b: float, a: float) -> float:
    """POBTASI of n blocks (the L^{-1} form)."""
    return (n - 1) * s_end(b, a) + 2 * b ** 3 / 3 + 2 * a * b * b + 2 * a * a * b + 2 * a ** 3 / 3


def reduced_blocks(P: int, scheme: str = "paper") -> int:
    if P <= 1:
        return 0
    return 2 * P - 1 if scheme == "paper" else 2 * P - 2


def balance_ratio(n: int, P: int, w_end: float, w_mid: float, scheme: str = "paper") -> float:
    """r = n_end / n_mid with equal work: (n_end - 1) w_end = (n_mid - 2) w_mid and
    n = e n_end + m n_mid (e end partitions of size n_end, m middle ones); the
    solution of the linear system, continuous in the sizes."""
    e, m = (1, P - 1) if scheme == "paper" else (2, P - 2)
    if m <= 0:
        return 1.0
    # n_end = (n_mid - 2) w_mid / w_end + 1  ->  e ((n_mid - 2) q + 1) + m n_mid = n, q = w_mid / w_end
    q = w_mid / w_end
    n_mid = (n - e + 2 * e * q) / (e * q + m)
    n_end = (n_mid - 2) * q + 1
    return n_end / n_mid


@dataclass
class LoadBalance:
    r_F: float
    r_S: float
    rho: float
    r_LB: float


def load_balance(n: int, P: int, b: float = 1024, a: float = 256, scheme: str = "paper") -> LoadBalance:
    """Table 4's quantities for this cost model: r_F (PPOBTAF), r_S (PPOBTASI), rho =
    PPOBTAF / PPOBTASI operations of the partitioned run, r_LB = rho r_F + (1-rho) r_S."""
    rF = balance_ratio(n, P, f_end(b, a), f_mid(b, a), scheme)
    rS = balance_ratio(n, P, s_end(b, a), s_mid(b, a), scheme)
    sizes = partition_sizes(n, P, 1.0, scheme)
    F = sum(_part_work(k, kind, b, a)[0] for k, kind in sizes)
    S = sum(_part_work(k, kind, b, a)[1] for k, kind in sizes)
    rho = F / S
    return LoadBalance(rF, rS, rho, weighted_r_lb(rF, rS, rho))


def weighted_r_lb(r_F: float, r_S: float, rho: float) -> float:
    """Reading SURVEY Q15 of Table 4's 'weighting the results with the number of
    operations performed for each function': r_LB = rho r_F + (1 - rho) r_S."""
    return rho * r_F + (1.0 - rho) * r_S


def partition_sizes(n: int, P: int, r: float, scheme: str = "paper"):
    """Continuous partition sizes for ratio r: [(size, kind)] with kind 'end' / 'mid'."""
    if P == 1:
        return [(float(n), "end")]
    e, m = (1, P - 1) if scheme == "paper" else (2, P - 2)
    n_mid = n / (e * r + m)
    out = [(r * n_mid, "end")] + [(n_mid, "mid")] * m
    if e == 2:
        out.append((r * n_mid, "end"))
    return out


def _part_work(k: float, kind: str, b: float, a: float):
    if kind == "end":
        return (k - 1) * f_end(b, a), (k - 1) * s_end(b, a)
    return (k - 2) * f_mid(b, a), (k - 2) * s_mid(b, a)


def efficiency(n: int, P: int, b: float = 1024, a: float = 256, r: float | None = None,
               scheme: str = "paper") -> tuple[float, float]:
    """(E, TFLOP per process): the theoretical maximum parallel efficiency of
    PPOBTAF + POBTARSSI + PPOBTASI (Sec. 4.4, Fig. 3a) at ratio r (default: the
    model's r_LB).  E = W_seq / (P W_proc)."""
    W_seq = f_seq(n, b, a) + s_seq(n, b, a)
    if P == 1:
        return 1.0, W_seq / 1e12
    if r is None:
        r = load_balance(n, P, b, a, scheme).r_LB
    busiest = max(sum(_part_work(k, kind, b, a)) for k, kind in partition_sizes(n, P, r, scheme))
    nr = reduced_blocks(P, scheme)
    W_proc = busiest + f_seq(nr, b, a) + s_seq(nr, b, a)
    return W_seq / (P * W_proc), W_proc / 1e12


# PAPER.md Table 4: n, load balancing PPOBTAF, PPOBTASI, ratio, r_LB
TABLE4 = [(32, 1.79, 2.43, 0.34, 2.22), (64, 1.83, 2.45, 0.34, 2.24), (128, 1.84, 2.46, 0.35, 2.24),
          (256, 1.85, 2.46, 0.35, 2.25), (512, 1.86, 2.46, 0.35, 2.25)]


def report(b: float = 1024, a: float = 256, ns=(32, 64, 128, 256, 512), Ps=(1, 2, 4, 8, 16, 32)) -> str:
    """Table 4 (paper vs this model) and the Fig. 3a efficiency grid, as text."""
    lines = [f"Load balancing (PAPER Table 4; b={b:g}, a={a:g}; model at P = 2, paper scheme)",
             "  n    paper r_F r_S  rho  r_LB | Q15(paper rows) | model r_F  r_S   rho   r_LB"]
    for n, rF, rS, rho, rLB in TABLE4:
        lb = load_balance(n, 2, b, a)
        lines.append(f"  {n:<4d} {rF:5.2f} {rS:5.2f} {rho:4.2f} {rLB:5.2f} | {weighted_r_lb(rF, rS, rho):15.3f} |"
                     f" {lb.r_F:9.2f} {lb.r_S:5.2f} {lb.rho:5.2f} {lb.r_LB:6.2f}")
    for scheme in ("paper", "twisted"):
        lines.append(f"Theoretical efficiency E(n, P) (Sec. 4.4 / Fig. 3a; scheme={scheme}; "
                     f"TFLOP per process in parentheses)")
        lines.append("  P\\n " + "".join(f"{n:>16d}" for n in ns))
        for P in Ps:
            row = []
            for n in ns:
                if P > 1 and n < 2 * P:
                    row.append(f"{'-':>16s}")
                    continue
                E, w = efficiency(n, P, b, a, scheme=scheme)
                row.append(f"{100 * E:8.1f}% ({w:5.2f})")
            lines.append(f"  {P:<4d}" + "".join(row))
    return "\n".join(lines)


if __name__ == "__main__":
    print(report())
