"""Multi-GPU step time from measured per-rank phases on ONE B200 (dev tool).

The GPU box has one B200, so the N-GPU distributed step (bench.py --gpus N:
serinv_ppobtaf -> NCCL all-gather -> serinv_ppobtasi) is
composed from its parts, each measured for real:

  * every rank's serinv_ppobtaf and serinv_ppobtasi graph runs ALONE on the
    whole GPU (as it would on its own B200), device-timed with CUDA events;
  * the all-gather is the only inter-GPU transfer: P records of
    serinv_exchange_bytes(b, a) each; modelled as a ring all-gather at
    BW_NVLINK bus bandwidth plus a fixed latency (both stated in the output).

  T(P) = max_p T_ppobtaf(p) + T_allgather(P) + max_p T_ppobtasi(p)

Weak scaling (C4: n = 256 per GPU): E(P) = T(1) / T(P), T(1) = the best
single-GPU step on n = 256 (sequential selinv or the library's intra-GPU plan,
both printed).  This is a model of the multi-GPU run composed of measured
parts, not a measurement of one; bench.py --gpus N measures the real thing.

    python tools/scaling_sim.py C4 1,2,4,8 [--r 1.0] [--strong]
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, "/root/repo")
import btagen  # noqa: E402
import paper_2503_17528_b200 as sb  # noqa: E402
from paper_2503_17528_b200 import distributed as sd  # noqa: E402

CFG = {"C2": (128, 1024, 64), "C3": (365, 2048, 4), "C4": (256, 512, 16), "C5": (16384, 64, 8)}
BW_NVLINK = 700e9      # assumed all-gather bus bandwidth per GPU on NVLink 5 (B/s)
LAT_ALLGATHER = 30e-6  # assumed fixed NCCL all-gather latency at P <= 8 (s)


def flops(n, b, a):
    F = (n - 1) * (7 / 3 * b**3 + 3 * a * b * b + a * a * b) + b**3 / 3 + a * b * b + a * a * b + a**3 / 3
    S = (n - 1) * (14 / 3 * b**3 + 6 * a * b * b + 2 * a * a * b) + 2 * b**3 / 3 + 2 * a * b * b + 2 * a * a * b + 2 * a**3 / 3
    return F + S


def timed(fn):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def single(n, b, a, Ps, reps):
    A0 = btagen.g1_torch(0, n, b, a)
    D = {k: v.clone() for k, v in A0.items()}
    best = float("inf")
    for _ in range(reps + 1):
        for k in D:
            D[k].copy_(A0[k])
        if Ps == [1]:
            t = timed(lambda: sb.selinv(D["diag"], D["lower"], D["arrow"], D["tip"], check=False))
        else:
            t = timed(lambda: sb.pselinv(D["diag"], D["lower"], D["arrow"], D["tip"], Ps, check=False))
        best = min(best, t)
    del A0, D
    torch.cuda.empty_cache()
    return best


def distributed(n, b, a, P, r, reps, q="auto"):
    """Per-rank phase times; one rank resident at a time (memory of one GPU)."""
    h = sb.default_handle()
    parts = sb.plan_ends(n, P, r)
    Q = sd.dist_auto_q(min(e - s for s, e in parts), b) if q == "auto" else int(q)

    inputs = {}

    def rank_state(p):
        s, e = parts[p]
        if p not in inputs:   # pristine rank inputs stay resident (the matrix once)
            A0 = btagen.g1_torch(0, n, b, a, start=s, end=e)
            if A0["lower"].shape[0] == 0:
                A0["lower"] = torch.zeros((1, b, b), dtype=torch.float64, device="cuda")
            inputs[p] = A0
        A0 = inputs[p]
        D = {k: v.clone() for k, v in A0.items()}
        return A0, D, sd.DistContext(h, P, p, n, s, e - s, b, a, Q=Q)

    def restore(A0, D):
        for k in D:
            D[k].copy_(A0[k])

    tF, tS, sends = [], [], []
    for p in range(P):          # pass 1: ppobtaf of every rank, keep its records
        A0, D, ctx = rank_state(p)
        best = float("inf")
        for _ in range(reps + 1):
            restore(A0, D)
            best = min(best, timed(lambda: sd.ppobtaf(ctx, D)))
        tF.append(best)
        sends.append(ctx.send.clone())
        del A0, D, ctx
        torch.cuda.empty_cache()
    recv = torch.cat(sends)
    del sends
    for p in range(P):          # pass 2: ppobtaf (untimed, rebuilds the workspace) + ppobtasi
        A0, D, ctx = rank_state(p)
        best = float("inf")
        for _ in range(reps + 1):
            restore(A0, D)
            sd.ppobtaf(ctx, D)
            ctx.recv.copy_(recv)
            best = min(best, timed(lambda: sd.ppobtasi(ctx, D)))
        if int(ctx.info.item()) != 0:
            raise SystemExit(f"info {int(ctx.info.item())}")
        tS.append(best)
        del A0, D, ctx
        torch.cuda.empty_cache()
    inputs.clear()
    torch.cuda.empty_cache()
    rec = sb.exchange_bytes(b, a)
    t_ag = LAT_ALLGATHER + (P - 1) * Q * rec / BW_NVLINK if P > 1 else 0.0
    return tF, tS, t_ag, parts, Q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("Ps")
    ap.add_argument("--r", type=float, default=1.0, help="end-rank ratio (bench default: distributed.auto_r(b))")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--strong", action="store_true", help="fixed total n (strong scaling)")
    ap.add_argument("--no-seq", action="store_true", help="skip the one-chain T1 when the auto plan partitions")
    ap.add_argument("--shape", default=None, help="n,b,a instead of a named config (e.g. dataset (1): 256,1024,256)")
    ap.add_argument("--q", default="auto", help="sub-partitions per rank, comma list (auto = serinv_dist_auto_q)")
    args = ap.parse_args()
    n1, b, a = CFG[args.config] if args.shape is None else map(int, args.shape.split(","))
    out = {"config": args.config, "b": b, "a": a, "r": args.r, "bw_allgather_model": BW_NVLINK,
           "lat_allgather_model": LAT_ALLGATHER, "rows": []}
    Pauto = sb.auto_partitions(n1, b)
    t_seq = single(n1, b, a, [1], args.reps) if (Pauto == [1] or not args.no_seq) else float("inf")
    t_auto = single(n1, b, a, Pauto, args.reps) if Pauto != [1] else t_seq
    t1 = min(t_seq, t_auto)
    out["T1"] = {"n": n1, "sequential_ms": round(t_seq * 1e3, 3), "auto_plan": Pauto,
                 "auto_ms": round(t_auto * 1e3, 3)}
    print(json.dumps(out["T1"]), flush=True)
    for P, q in [(int(x), q) for x in args.Ps.split(",") for q in args.q.split(",")]:
        if P == 1:
            continue
        n = n1 if args.strong else n1 * P
        try:
            tF, tS, t_ag, parts, Q = distributed(n, b, a, P, args.r, args.reps, q)
        except RuntimeError as ex:
            print(json.dumps({"P": P, "q": q, "error": str(ex)}), flush=True)
            continue
        T = max(tF) + t_ag + max(tS)
        # flop-model ceiling: sequential work / (P x (busiest rank + redundant reduced solve));
        # per block F+SI ~ 7 b^3 at the chain ends, ~19 b^3 in a middle partition (fill-in chains)
        w_rank = []
        for p, (s_, e_) in enumerate(parts):
            c = e_ - s_
            subs = [c // Q + (1 if q < c % Q else 0) for q in range(Q)]
            w_rank.append(sum((7 if (p * Q + q in (0, P * Q - 1)) else 19) * m for q, m in enumerate(subs)))
        w_red = 7 * (2 * P * Q - 2)
        e_flop = 7 * n / (P * (max(w_rank) + w_red))
        row = {"E_flop_model": round(e_flop, 4),"P": P, "Q": Q, "n": n, "parts": parts, "ppobtaf_ms": [round(x * 1e3, 3) for x in tF],
               "ppobtasi_ms": [round(x * 1e3, 3) for x in tS], "allgather_ms_model": round(t_ag * 1e3, 4),
               "T_ms": round(T * 1e3, 3), "TFLOPs_total": round(flops(n, b, a) / T / 1e12, 3),
               ("E_strong" if args.strong else "E_weak"): round(t1 / (P * T) if args.strong else t1 / T, 4)}
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
