"""SERINV_OPT knob sweep of the fused selinv step (dev tool; the graph cache is keyed by
the option string, so one process can time several settings).

    python tools/knobs.py C3 "" "urgent_ctas=4" "fuse_trsm3=1,urgent_ctas=2"
"""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import btagen  # noqa: E402
import paper_2503_17528_b200 as sb  # noqa: E402
from bench import CONFIGS, flops_pobtaf, flops_pobtasi  # noqa: E402


def main():
    cfg = sys.argv[1]
    n, b, a = CONFIGS[cfg]["n"], CONFIGS[cfg]["b"], CONFIGS[cfg]["a"]
    fl = flops_pobtaf(n, b, a) + flops_pobtasi(n, b, a)
    A0 = btagen.g1_torch(0, n, b, a)
    D = {k: v.clone() for k, v in A0.items()}
    for opt in sys.argv[2:]:
        os.environ["SERINV_OPT"] = opt
        t0 = time.time()
        sb.graph_stats(2, n, b, a)
        tb = time.time() - t0
        ts = []
        for r in range(5):
            for k in D:
                D[k].copy_(A0[k])
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            sb.selinv(D["diag"], D["lower"], D["arrow"], D["tip"], check=False)
            e1.record()
            torch.cuda.synchronize()
            if r >= 1:
                ts.append(e0.elapsed_time(e1))
        med = statistics.median(ts)
        print(f"{cfg} opt='{opt}': {med:.2f} ms  {fl / med / 1e9:.2f} TFLOP/s  (build {tb:.1f}s)", flush=True)


if __name__ == "__main__":
    main()
