"""Executor utilisation over time from one traced launch (dev tool).

    python tools/utilization.py selinv 365 2048 4 [--bins 40]

Per time bin: the share of CTA-time spent executing tasks (start..end), waiting on
dependencies (claim..start) and idle (between tasks / after the CTA's queue
drained), plus the DMMA flops executed by type; the time of the last POTRF (end of
the factorisation chain) and the executed-flop rate per phase.
"""
import argparse
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import btagen  # noqa: E402
import paper_2503_17528_b200 as sb  # noqa: E402
from paper_2503_17528_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind")
    ap.add_argument("n", type=int)
    ap.add_argument("b", type=int)
    ap.add_argument("a", type=int)
    ap.add_argument("--bins", type=int, default=40)
    args = ap.parse_args()
    n, b, a = args.n, args.b, args.a
    kid = {"selinv": 2, "pobtaf": 0, "pobtasi": 1}[args.kind]
    h = sb.default_handle()
    st = sb.graph_stats(kid, n, b, a)
    T = st["tasks"]
    grid = st["grid"]
    L = _lib.lib()
    D = btagen.g1_torch(0, n, b, a)
    buf = torch.zeros(12 * T, dtype=torch.int64, device="cuda")
    L.serinv_set_trace(h._h, buf.data_ptr(), buf.numel() * 8)
    fn = {"selinv": sb.selinv, "pobtaf": sb.pobtaf, "pobtasi": sb.pobtasi}[args.kind]
    for _ in range(2):
        Dc = {k: v.clone() for k, v in D.items()}
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(Dc["diag"], Dc["lower"], Dc["arrow"], Dc["tip"], check=False)
        e1.record()
        torch.cuda.synchronize()
        print("launch ms (traced)", round(e0.elapsed_time(e1), 3))
    L.serinv_set_trace(h._h, None, 0)
    tr = buf[:4 * T].view(T, 4).cpu().numpy().astype(np.int64)
    claim, start, end, meta = tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 3]
    ok = end > 0
    t0 = claim[ok].min()
    claim, start, end = claim - t0, start - t0, end - t0
    typ = meta & 0xFFFF
    sm = (meta >> 16) & 0xFFFF
    mm = (meta >> 32) & 0xFFFF
    flg = (meta >> 48) & 0xFFFF
    span = end[ok].max()
    print(f"tasks {T} grid {grid} makespan {span / 1e6:.3f} ms")
    names = {1: "GEMM", 2: "POTRF", 3: "TRTRI", 4: "REDUCE", 5: "COPY", 6: "LOGDET"}
    for t, nm in names.items():
        sel = ok & (typ == t)
        if sel.any():
            d = (end[sel] - start[sel]) / 1e3
            w = (start[sel] - claim[sel]) / 1e3
            print(f"  {nm:7s} count {sel.sum():8d}  exec {d.sum() / 1e3:10.2f} ms-CTA (mean {d.mean():7.2f} us)"
                  f"  wait {w.sum() / 1e3:10.2f} ms-CTA (mean {w.mean():7.2f} us)")
    wide = ok & (typ == 1) & (mm > 64)
    if wide.any():
        print(f"  wide GEMM tasks {wide.sum()} exec mean {((end[wide] - start[wide]) / 1e3).mean():.2f} us")
    last_potrf = end[ok & (typ == 2)].max() if (ok & (typ == 2)).any() else 0
    print(f"last POTRF ends at {last_potrf / 1e6:.3f} ms ({100 * last_potrf / span:.1f} % of the makespan)")
    # per-bin occupancy: exec / wait / idle of grid CTA slots
    bins = args.bins
    edges = np.linspace(0, span, bins + 1)
    ex = np.zeros(bins)
    wt = np.zeros(bins)

    def add(acc, a0, a1):
        for i in range(bins):
            lo, hi = edges[i], edges[i + 1]
            ov = np.clip(np.minimum(a1, hi) - np.maximum(a0, lo), 0, None)
            acc[i] += ov.sum()

    add(ex, start[ok], end[ok])
    add(wt, claim[ok], start[ok])
    width = span / bins
    print(f"{'t ms':>8s} {'exec%':>6s} {'wait%':>6s} {'idle%':>6s}")
    for i in range(bins):
        e = 100 * ex[i] / (grid * width)
        w = 100 * wt[i] / (grid * width)
        print(f"{edges[i] / 1e6:8.2f} {e:6.1f} {w:6.1f} {100 - e - w:6.1f}")
    print(f"overall: exec {100 * ex.sum() / (grid * span):.1f} %  wait {100 * wt.sum() / (grid * span):.1f} %")
    _ = (sm, flg)


if __name__ == "__main__":
    main()
