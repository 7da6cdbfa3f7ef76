"""Time the in-process partitioned pipeline (serinv_pselinv) on the bench configs under
several partition counts (dev tool): python tools/pselinv_plans.py"""
import sys, statistics, torch
sys.path.insert(0, "/root/repo")
import btagen, paper_2503_17528_b200 as sb
from bench import CONFIGS, flops_pobtaf, flops_pobtasi
for cfg, plans in (("C2", [[2], [3], [4]]), ("C3", [[2], [3]]), ("C4", [[4], [3], [6], [8]])):
    n, b, a = CONFIGS[cfg]["n"], CONFIGS[cfg]["b"], CONFIGS[cfg]["a"]
    fl = flops_pobtaf(n, b, a) + flops_pobtasi(n, b, a)
    A0 = btagen.g1_torch(0, n, b, a)
    D = {k: v.clone() for k, v in A0.items()}
    print(cfg, "auto", sb.auto_partitions(n, b), flush=True)
    for Ps in plans:
        ts = []
        for r in range(5):
            for k in D: D[k].copy_(A0[k])
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); sb.pselinv(D["diag"], D["lower"], D["arrow"], D["tip"], Ps, check=(r == 0)); e1.record()
            torch.cuda.synchronize()
            if r >= 1: ts.append(e0.elapsed_time(e1))
        m = statistics.median(ts)
        print(cfg, Ps, f"{m:.2f} ms {fl/m/1e9:.2f} TFLOP/s", flush=True)
