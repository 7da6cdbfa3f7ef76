"""Per-kernel device times of one library call (dev tool; torch.profiler / CUPTI).

    python tools/kernel_times.py sb 16384 64 8            # small-block engine, library plan
    python tools/kernel_times.py selinv 365 2048 4
"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, "/root/repo")
import btagen  # noqa: E402
import paper_2503_17528_b200 as sb  # noqa: E402


def main():
    kind, n, b, a = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    Ps = None if len(sys.argv) < 6 else [int(x) for x in sys.argv[5].split("x")]
    A = btagen.g1_torch(0, n, b, a)

    def call():
        D = {k: v.clone() for k, v in A.items()}
        torch.cuda.synchronize()
        if kind == "sb":
            sb.selinv_sb(D["diag"], D["lower"], D["arrow"], D["tip"], Ps, check=False)
        else:
            sb.selinv(D["diag"], D["lower"], D["arrow"], D["tip"], check=False)
        torch.cuda.synchronize()

    for _ in range(3):
        call()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        call()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and ("sb_" in e.name or "serinv" in e.name)]
    tot = 0.0
    for e in evs:
        us = e.device_time if hasattr(e, "device_time") else e.cuda_time
        tot += us
        print(f"{e.name[:40]:40s} {us:10.1f} us")
    print(f"total {tot:.1f} us; plan {sb.sb_auto_plan(n, b, a) if kind == 'sb' and Ps is None else Ps}")


if __name__ == "__main__":
    main()
