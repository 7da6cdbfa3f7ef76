"""Quick device timing of selinv / pobtaf / pobtasi on one shape (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '/root/repo')
import btagen
import paper_2503_17528_b200 as sb

def main(n, b, a, reps=3, kinds=("selinv", "pobtaf")):
    A = btagen.g1(0, n, b, a)
    D0 = {k: torch.from_numpy(A[k]).cuda() for k in ("diag", "lower", "arrow", "tip")}
    D = {k: v.clone() for k, v in D0.items()}
    args = (D["diag"], D["lower"], D["arrow"], D["tip"])
    F = (n - 1) * (7 / 3 * b**3 + 3 * a * b * b + a * a * b) + b**3 / 3 + a * b * b + a * a * b + a**3 / 3
    S = (n - 1) * (14 / 3 * b**3 + 6 * a * b * b + 2 * a * a * b) + 2 * b**3 / 3 + 2 * a * b * b + 2 * a * a * b + 2 * a**3 / 3
    h = sb.default_handle()
    t0 = time.time(); sb.graph_stats(2, n, b, a); sb.graph_stats(0, n, b, a); print("graph build s", time.time() - t0, flush=True)
    for kind in kinds:
        fn = getattr(sb, kind)
        fl = F + S if kind == "selinv" else F
        for r in range(reps):
            for k in D: D[k].copy_(D0[k])
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(*args, check=False)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            print(kind, n, b, a, f"{ms:.2f} ms", f"{fl / ms / 1e9:.2f} TFLOP/s", "info", int(h.scalars()[0].item()), "logdet", float(h.scalars()[1].item()), flush=True)

if __name__ == "__main__":
    n, b, a = map(int, sys.argv[1:4])
    main(n, b, a)
