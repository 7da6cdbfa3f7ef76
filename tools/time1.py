"""Device time of one config (dev tool): python tools/time1.py C2 [P|auto] [reps].
Options come from SERINV_OPT (graph build), so sweeps run one process per setting."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import btagen
import paper_2503_17528_b200 as sb
from tools.sweep import CFG, flops

name = sys.argv[1]
P = sys.argv[2] if len(sys.argv) > 2 else "1"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
r = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
n, b, a = CFG[name]
Ps = sb.auto_partitions(n, b) if P == "auto" else [int(x) for x in P.split("x")]
A0 = btagen.g1_torch(0, n, b, a)
D = {k: v.clone() for k, v in A0.items()}
ts = []
for it in range(reps + 1):
    for k in D:
        D[k].copy_(A0[k])
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    if Ps == [1]:
        sb.selinv(D["diag"], D["lower"], D["arrow"], D["tip"], check=False)
    else:
        sb.pselinv(D["diag"], D["lower"], D["arrow"], D["tip"], Ps, r, check=False)
    e1.record(); torch.cuda.synchronize()
    if it:
        ts.append(e0.elapsed_time(e1))
ms = min(ts)
print(f"{name} P={P} r={r} opt={os.environ.get('SERINV_OPT', '')}: {ms:.2f} ms {flops(n, b, a) / ms / 1e9:.2f} TF/s (all {[round(t, 2) for t in ts]})", flush=True)
