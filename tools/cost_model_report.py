"""Analytic cost model (paper_2503_17528_b200/costmodel.py: Table 4 r_LB, Sec. 4.4
efficiency grid) printed next to the round-1 composed step model measured on one B200
(profiles/r01/dataset1/: per-rank launches timed alone, all-gather modelled).

    python tools/cost_model_report.py > profiles/r02/costmodel.txt
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2503_17528_b200 import costmodel as cm  # noqa: E402

print(cm.report())
print()
print("Dataset (1) (b=1024, a=256) strong scaling: flop model vs the composed step model measured on one B200")
print("(profiles/r01/dataset1; E_strong = T_1 / (P T_P), T_P = max ppobtaf + all-gather model + max ppobtasi;")
print(" twisted scheme, r = 1, Q sub-partitions per rank as measured)")
print("  n     P  Q   E_model(twisted, r_LB)  E_model(twisted, r=1)  E_measured")
for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r01", "dataset1", "d1_n*.txt")),
                key=lambda p: int(p.split("_n")[1].split(".")[0])):
    with open(f) as fh:
        rows = [json.loads(line) for line in fh if line.startswith("{\"E_flop")]
    for r in rows:
        n, P = r["n"], r["P"]
        e1 = cm.efficiency(n, P, scheme="twisted")[0]
        e2 = cm.efficiency(n, P, r=1.0, scheme="twisted")[0]
        print(f"  {n:<5d} {P:<2d} {r['Q']:<2d}  {100 * e1:20.1f}%  {100 * e2:20.1f}%  {100 * r['E_strong']:9.1f}%")
