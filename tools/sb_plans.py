"""Time the small-block engine on one shape under several nesting plans (dev tool).

    python tools/sb_plans.py 16384 64 8 auto 148x74x37x18x9x4 148x74x37x18x9x2
"""
import statistics
import sys

import torch

sys.path.insert(0, "/root/repo")
import btagen  # noqa: E402
import paper_2503_17528_b200 as sb  # noqa: E402


def main():
    n, b, a = (int(x) for x in sys.argv[1:4])
    A0 = btagen.g1_torch(0, n, b, a)
    D = {k: v.clone() for k, v in A0.items()}
    fl = ((n - 1) * (7 / 3 * b ** 3 + 3 * a * b * b + a * a * b) + b ** 3 / 3 + a * b * b + a * a * b + a ** 3 / 3
          + (n - 1) * (14 / 3 * b ** 3 + 6 * a * b * b + 2 * a * a * b) + 2 * b ** 3 / 3 + 2 * a * b * b
          + 2 * a * a * b + 2 * a ** 3 / 3)
    for spec in sys.argv[4:]:
        Ps = sb.sb_auto_plan(n, b, a) if spec == "auto" else [int(x) for x in spec.split("x")]
        ts = []
        ld = None
        for r in range(7):
            for k in D:
                D[k].copy_(A0[k])
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            out = sb.selinv_sb(D["diag"], D["lower"], D["arrow"], D["tip"], Ps, check=r == 0)
            if r == 0:
                ld = out
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        med = statistics.median(ts)
        print(f"plan {'x'.join(map(str, Ps)):28s} {med:.3f} ms  {fl / med / 1e9:.2f} TFLOP/s  logdet {ld:.6f}", flush=True)


if __name__ == "__main__":
    main()
