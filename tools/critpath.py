"""Binding dependencies of the critical chain (dev tool): runs one traced launch,
then for every POTRF / chain-TRSM task reports which producer finished last
before it could start (the dependency that bound it) and the slack.

    python tools/critpath.py selinv 128 1024 64
"""
import ctypes, sys, collections
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import btagen
import paper_2503_17528_b200 as sb
from paper_2503_17528_b200 import _lib

NAMES = {1: "GEMM", 2: "POTRF", 3: "TRTRI", 4: "REDUCE", 5: "COPY", 6: "LOGDET"}


def role(t, f, q):
    if t == 1:
        if f & 256: return "CHAIN_TS"
        if f & 2: return "TRSM"
        if f & 1: return "GEMM_MIR"
        return "UPDATE"
    return NAMES.get(int(t), str(t)) + (f"/q{q}" if q else "")


def main():
    kind, n, b, a = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    kid = {"selinv": 2, "pobtaf": 0}[kind]
    h = sb.default_handle()
    st = sb.graph_stats(kid, n, b, a)
    T = st["tasks"]
    L = _lib.lib()
    nw, ns = ctypes.c_int64(0), ctypes.c_int64(0)
    L.serinv_graph_dump.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                    ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
    assert L.serinv_graph_dump(h._h, kid, n, b, a, 1, 1.0, None, None, ctypes.byref(nw), None, ctypes.byref(ns)) == 0
    rec = np.zeros((T, 10), np.int32); waits = np.zeros(nw.value, np.int32); sigs = np.zeros(ns.value, np.int32)
    assert L.serinv_graph_dump(h._h, kid, n, b, a, 1, 1.0, rec.ctypes.data, waits.ctypes.data, None,
                               sigs.ctypes.data, None) == 0
    D = btagen.g1_torch(0, n, b, a)
    buf = torch.zeros(12 * T, dtype=torch.int64, device="cuda")
    L.serinv_set_trace(h._h, buf.data_ptr(), buf.numel() * 8)
    fn = {"selinv": sb.selinv, "pobtaf": sb.pobtaf}[kind]
    for rep in range(2):
        Dc = {k: v.clone() for k, v in D.items()}
        torch.cuda.synchronize()
        fn(Dc["diag"], Dc["lower"], Dc["arrow"], Dc["tip"], check=False)
        torch.cuda.synchronize()
    L.serinv_set_trace(h._h, None, 0)
    tr = buf[:4 * T].view(T, 4).cpu().numpy().astype(np.int64)
    claim, start, end = tr[:, 0], tr[:, 1], tr[:, 2]
    t0 = claim.min(); claim, start, end = claim - t0, start - t0, end - t0
    # producers per counter
    prod = collections.defaultdict(list)
    for t in range(T):
        for s in sigs[rec[t, 7]:rec[t, 7] + rec[t, 8]]:
            prod[int(s)].append(t)
    typ, fl, q = rec[:, 0], rec[:, 1], rec[:, 9]
    chain = [t for t in range(T) if q[t] in (1, 2, 3, 4) and typ[t] in (1, 2)]
    chain.sort(key=lambda t: start[t])
    stats = collections.defaultdict(list)
    for t in chain:
        ws = waits[rec[t, 4]:rec[t, 4] + rec[t, 5] - rec[t, 6]]  # early waits
        best, bp = -1, -1
        for c in ws:
            for p in prod[int(c)]:
                if end[p] > best:
                    best, bp = end[p], p
        if bp < 0:
            continue
        key = (role(typ[t], fl[t], q[t]), role(typ[bp], fl[bp], q[bp]))
        stats[key].append((start[t] - best, start[t] - claim[t], end[t] - start[t]))
    print(f"tasks {T}, chain tasks {len(chain)}, makespan {end.max() / 1e6:.2f} ms")
    print(f"{'task':14s} {'bound by':14s} {'count':>6s} {'gap us':>8s} {'waited us':>10s} {'dur us':>8s}")
    for key, v in sorted(stats.items(), key=lambda kv: -len(kv[1])):
        v = np.array(v) / 1e3
        print(f"{key[0]:14s} {key[1]:14s} {len(v):6d} {v[:, 0].mean():8.2f} {v[:, 1].mean():10.2f} {v[:, 2].mean():8.2f}")
    # timeline of a few consecutive chain steps (queues 1 and 2), relative to the first
    ph = buf[4 * T:].view(T, 8).cpu().numpy().astype(np.int64) - t0
    sel = [t for t in chain if q[t] in (1, 2)]
    sel.sort(key=lambda t: start[t])
    mid = len(sel) // 2
    base = claim[sel[mid]]
    print("timeline (us, relative): queue role claim start [phases] end")
    for t in sel[mid:mid + 8]:
        p = [f"{(v - base) / 1e3:7.2f}" for v in ph[t] if v > 0]
        print(f"  q{q[t]} {role(typ[t], fl[t], q[t]):10s} {(claim[t] - base) / 1e3:7.2f} {(start[t] - base) / 1e3:7.2f} "
              f"[{' '.join(p)}] {(end[t] - base) / 1e3:7.2f}")
    # period of each critical queue
    for qq in (1, 2, 3, 4):
        sel = [t for t in chain if q[t] == qq]
        if len(sel) > 2:
            e = np.sort(end[sel])
            print(f"queue {qq}: {len(sel)} tasks, period {np.diff(e).mean() / 1e3:.2f} us, busy {((end - start)[sel]).sum() / (e[-1] - e[0]):.2f}")


if __name__ == "__main__":
    main()
