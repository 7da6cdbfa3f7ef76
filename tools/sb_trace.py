"""Phase timestamps of the small-block engine (dev tool): one middle partition per level.

    python tools/sb_trace.py 16384 64 8 [148x49x16x5]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import btagen  # noqa: E402
import paper_2503_17528_b200 as sb  # noqa: E402
from paper_2503_17528_b200 import _lib  # noqa: E402


def chol_rounds(buf, lvl, k):
    """chol_inv64 internal stamps of step k at level lvl (factor kernel, traced partition)."""
    t = buf.view(-1).cpu().numpy().astype(np.int64)
    base = ((8 + lvl) * 2 * 128 + 2 * k) * 8
    return t[base:base + 16]


def main():
    n, b, a = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    Ps = sb.sb_auto_plan(n, b, a) if len(sys.argv) < 5 else [int(x) for x in sys.argv[4].split("x")]
    A = btagen.g1_torch(0, n, b, a)
    h = sb.default_handle()
    words = 16 * 2 * 128 * 8
    buf = torch.zeros(words + 64, dtype=torch.int64, device="cuda")
    for _ in range(2):
        D = {k: v.clone() for k, v in A.items()}
        sb.selinv_sb(D["diag"], D["lower"], D["arrow"], D["tip"], Ps, check=False)
    _lib.lib().serinv_set_trace(h._h, buf.data_ptr(), buf.numel() * 8)
    D = {k: v.clone() for k, v in A.items()}
    sb.selinv_sb(D["diag"], D["lower"], D["arrow"], D["tip"], Ps, check=False, handle=h)
    torch.cuda.synchronize()
    _lib.lib().serinv_set_trace(h._h, None, 0)
    t = buf[:words].view(16, 2, 128, 8).cpu().numpy().astype(np.int64)
    names = [["chol", "loads+W st", "TRSMs", "Schur"], ["loads", "Lc~ Lf~ Lam", "X_k+1,k Q X_nk", "X_kk"]]
    print(f"plan {Ps}")
    for lvl in range(len(Ps) + 1):
        for kern in range(2):
            T = t[lvl, kern]
            steps = [k for k in range(128) if T[k, 0] and T[k, 4]]
            if not steps:
                continue
            d = np.array([[T[k, i + 1] - T[k, i] for i in range(4)] for k in steps]) / 1e3
            tot = (T[steps, 4] - T[steps, 0]) / 1e3
            parts = "  ".join(f"{names[kern][i]} {d[:, i].mean():6.2f}" for i in range(4))
            print(f"level {lvl} {'factor ' if kern == 0 else 'inverse'} steps {len(steps):3d}  "
                  f"step {tot.mean():6.2f} us:  {parts}")
            if kern == 0 and lvl < 8:
                # chol_inv64 rounds: leaf(+copy) and trailing phases, then the W = L^{-1} phase
                rows = []
                for k in steps[:16]:
                    c = chol_rounds(buf, lvl, k)
                    t0 = T[k, 0]
                    if not c[15]:
                        continue
                    ev = [t0] + [c[i] for i in range(15)] + [c[15]]
                    rows.append(np.diff(np.array(ev, dtype=np.int64)) / 1e3)
                if rows:
                    r = np.array(rows).mean(axis=0)
                    print("    chol: " + " ".join(f"{x:5.2f}" for x in r) + "  (leaf_j trail_j ..., leaf_7, W)")


if __name__ == "__main__":
    main()

