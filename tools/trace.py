"""Per-task trace of one serinv launch (dev tool): where the time goes.

    python tools/trace.py selinv 128 1024 64 [--out gpurun_out/trace.npz]
"""
import argparse, ctypes, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import btagen
import paper_2503_17528_b200 as sb
from paper_2503_17528_b200 import _lib

NAMES = {1: "GEMM", 2: "POTRF", 3: "TRTRI", 4: "REDUCE", 5: "COPY", 6: "LOGDET", 11: "CHAIN_TS", 12: "TRSM", 13: "GEMM_MIR"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind")
    ap.add_argument("n", type=int); ap.add_argument("b", type=int); ap.add_argument("a", type=int)
    ap.add_argument("--P", default="1", help="partitions; nested as 256x16; 'auto'")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    n, b, a = args.n, args.b, args.a
    D = btagen.g1_torch(0, n, b, a)
    h = sb.default_handle()
    kindid = {"pobtaf": 0, "pobtasi": 1, "selinv": 2, "pselinv": 3}[args.kind]
    args.P = sb.auto_partitions(n, b) if args.P == "auto" else [int(x) for x in args.P.split("x")]
    if len(args.P) == 1:
        args.P = args.P[0]
    st = sb.graph_stats(kindid, n, b, a, args.P)
    T = st["tasks"]
    buf = torch.zeros(12 * T, dtype=torch.int64, device="cuda")
    _lib.lib().serinv_set_trace(h._h, buf.data_ptr(), buf.numel() * 8)
    fn = {"pobtaf": sb.pobtaf, "selinv": sb.selinv, "pobtasi": sb.pobtasi}.get(args.kind)
    for rep in range(2):
        Dc = {k: v.clone() for k, v in D.items()}
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        if args.kind == "pselinv":
            sb.pselinv(Dc["diag"], Dc["lower"], Dc["arrow"], Dc["tip"], args.P, check=False)
        else:
            fn(Dc["diag"], Dc["lower"], Dc["arrow"], Dc["tip"], check=False)
        e1.record(); torch.cuda.synchronize()
        print("launch ms", e0.elapsed_time(e1))
    _lib.lib().serinv_set_trace(h._h, None, 0)
    tr = buf[:4 * T].view(T, 4).cpu().numpy().astype(np.int64)
    ph = buf[4 * T:].view(T, 8).cpu().numpy().astype(np.int64)
    claim, start, end, meta = tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 3]
    t0 = claim.min()
    claim, start, end = claim - t0, start - t0, end - t0
    typ = meta & 0xFFFF; sm = (meta >> 16) & 0xFFFF; m = (meta >> 32) & 0xFFFF; fl = (meta >> 48) & 0xFFFF
    nn = fl
    # split GEMM by role: TRSM (post-multiply), chain TRSM+SYRK, mirrored (X_ii), other
    typ = typ.copy()
    typ[(typ == 1) & ((fl & 256) != 0)] = 11   # chain TRSM + SYRK
    typ[(typ == 1) & ((fl & 2) != 0)] = 12     # TRSM / W-post
    typ[(typ == 1) & ((fl & 1) != 0)] = 13     # mirrored X_ii
    span = end.max()
    print(f"tasks {T} makespan {span/1e6:.3f} ms  grid {st['grid']}  GF {st['flops']/1e9:.1f}")
    busy = (end - start).sum(); waited = (start - claim).sum()
    print(f"busy CTA-time {busy/1e6:.1f} ms, waiting CTA-time {waited/1e6:.1f} ms, capacity {st['grid']*span/1e6:.1f} ms")
    for t in sorted(set(typ.tolist())):
        sel = typ == t
        d = (end - start)[sel]; w = (start - claim)[sel]
        print(f"  {NAMES.get(t, t):7s} n={sel.sum():7d}  dur mean {d.mean()/1e3:7.2f} us  p50 {np.median(d)/1e3:7.2f}  p90 {np.percentile(d,90)/1e3:7.2f}  wait mean {w.mean()/1e3:7.2f} us  total {d.sum()/1e6:8.2f} ms")
    pot = np.where(typ == 2)[0]
    if len(pot) > 2:
        ends = np.sort(end[pot]); starts = np.sort(start[pot])
        gaps = np.diff(ends)
        print(f"  POTRF end-to-end period: mean {gaps.mean()/1e3:.2f} us p50 {np.median(gaps)/1e3:.2f} us  (x{len(pot)})")
        dur = (end - start)[pot]
        print(f"  POTRF duration mean {dur.mean()/1e3:.2f} us; claim->start {(start-claim)[pot].mean()/1e3:.2f} us")
        P_ = ph[pot] - t0
        st_ = start[pot]
        names = ["gemm(both)", "chol", "trtri", "trsm2", "store L,W"]
        prev = st_
        for k in range(5):
            cur = P_[:, k]
            ok = ph[pot][:, k] > 0
            if ok.any():
                print(f"    phase {names[k]:12s} {np.mean((cur - prev)[ok])/1e3:8.2f} us")
                prev = np.where(ok, cur, prev)

    pot_sms = set(sm[typ == 2].tolist())
    shared = int(((typ != 2) & np.isin(sm, list(pot_sms))).sum())
    print(f"  POTRF ran on SMs {sorted(pot_sms)[:8]}; GEMM tasks on those SMs: {shared}")
    # timeline utilisation in 10 buckets
    nb = 20
    edges = np.linspace(0, span, nb + 1)
    util = []
    for i in range(nb):
        lo, hi = edges[i], edges[i + 1]
        ov = np.clip(np.minimum(end, hi) - np.maximum(start, lo), 0, None).sum()
        util.append(ov / (st['grid'] * (hi - lo)))
    print("  utilisation per 5% of time:", " ".join(f"{u:.2f}" for u in util))
    # the least-utilised 5% window (before the last one): what runs, what waits
    k = int(np.argmin(util[:-1]))
    lo, hi = edges[k], edges[k + 1]
    run_ = (start < hi) & (end > lo)
    wait_ = (claim < hi) & (start > lo)
    print(f"  dip window {k}: {lo/1e6:.2f}-{hi/1e6:.2f} ms, util {util[k]:.2f}")
    for t in sorted(set(typ[run_ | wait_].tolist())):
        print(f"    {NAMES.get(t, t):8s} running {int((run_ & (typ == t)).sum()):6d}  claimed-waiting {int((wait_ & (typ == t)).sum()):6d}")
    pw = np.where(wait_ & (typ == 2))[0]
    if len(pw):
        print(f"    POTRF in window: rows(m) {sorted(set(m[pw].tolist()))[:5]} start-claim {((start - claim)[pw]).mean()/1e3:.1f} us")
    if args.out:
        np.savez(args.out, claim=claim, start=start, end=end, typ=typ, sm=sm, m=m, n=nn)


if __name__ == "__main__":
    main()
