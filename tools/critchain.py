"""Dependency chain behind the critical chain tasks, several levels deep (dev tool).

    python tools/critchain.py selinv 365 2048 4 [--depth 4] [--steps 3]

For a few consecutive chain tasks in the middle of the launch, walks back through
the producer that finished last among each task's early waits and prints every
task on that path: role, queue, claim / start / end (us, relative) and its size.
"""
import argparse
import collections
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import btagen  # noqa: E402
import paper_2503_17528_b200 as sb  # noqa: E402
from paper_2503_17528_b200 import _lib  # noqa: E402
from tools.critpath import role  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind")
    ap.add_argument("n", type=int)
    ap.add_argument("b", type=int)
    ap.add_argument("a", type=int)
    ap.add_argument("--depth", type=int, default=4)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    kid = {"selinv": 2, "pobtaf": 0}[args.kind]
    n, b, a = args.n, args.b, args.a
    h = sb.default_handle()
    T = sb.graph_stats(kid, n, b, a)["tasks"]
    L = _lib.lib()
    nw, ns = ctypes.c_int64(0), ctypes.c_int64(0)
    L.serinv_graph_dump.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
    assert L.serinv_graph_dump(h._h, kid, n, b, a, 1, 1.0, None, None, ctypes.byref(nw), None, ctypes.byref(ns)) == 0
    rec = np.zeros((T, 10), np.int32)
    waits = np.zeros(nw.value, np.int32)
    sigs = np.zeros(ns.value, np.int32)
    assert L.serinv_graph_dump(h._h, kid, n, b, a, 1, 1.0, rec.ctypes.data, waits.ctypes.data, None,
                               sigs.ctypes.data, None) == 0
    D = btagen.g1_torch(0, n, b, a)
    buf = torch.zeros(12 * T, dtype=torch.int64, device="cuda")
    L.serinv_set_trace(h._h, buf.data_ptr(), buf.numel() * 8)
    fn = {"selinv": sb.selinv, "pobtaf": sb.pobtaf}[args.kind]
    for _ in range(2):
        Dc = {k: v.clone() for k, v in D.items()}
        torch.cuda.synchronize()
        fn(Dc["diag"], Dc["lower"], Dc["arrow"], Dc["tip"], check=False)
        torch.cuda.synchronize()
    L.serinv_set_trace(h._h, None, 0)
    tr = buf[:4 * T].view(T, 4).cpu().numpy().astype(np.int64)
    claim, start, end, meta = tr[:, 0], tr[:, 1], tr[:, 2], tr[:, 3]
    prod = collections.defaultdict(list)
    for t in range(T):
        for sg in sigs[rec[t, 7]:rec[t, 7] + rec[t, 8]]:
            prod[int(sg)].append(t)
    typ, fl, q = rec[:, 0], rec[:, 1], rec[:, 9]
    chain = sorted([t for t in range(T) if q[t] in (1, 2) and typ[t] in (1, 2)], key=lambda t: start[t])
    mid = len(chain) // 2
    base = claim[chain[mid]]
    mm = (meta >> 32) & 0xFFFF

    def binding(t):
        ws = waits[rec[t, 4]:rec[t, 4] + rec[t, 5] - rec[t, 6]]
        best, bp = -1, -1
        for c in ws:
            for p in prod[int(c)]:
                if end[p] > best:
                    best, bp = end[p], p
        return bp

    for t in chain[mid:mid + args.steps]:
        print(f"--- chain task {t}")
        cur, d = t, 0
        while cur >= 0 and d <= args.depth:
            print(f"  {'  ' * d}{role(typ[cur], fl[cur], q[cur]):10s} q{q[cur]} m={mm[cur]:3d} "
                  f"claim {(claim[cur] - base) / 1e3:9.2f} start {(start[cur] - base) / 1e3:9.2f} "
                  f"end {(end[cur] - base) / 1e3:9.2f} (dur {(end[cur] - start[cur]) / 1e3:6.2f}, "
                  f"waited {(start[cur] - claim[cur]) / 1e3:6.2f}) nwait {rec[cur, 5]} nlate {rec[cur, 6]}")
            cur = binding(cur)
            d += 1


if __name__ == "__main__":
    main()
