"""Per-kernel SASS instruction histogram of libserinv.so (dev tool; no GPU needed).

    python tools/sass_hist.py > profiles/r02/sass_histogram.txt

Counts static instructions by opcode (the mnemonic before the first '.') for every
kernel, and lists the FP64 tensor / memory-movement opcodes that prove the data path:
DMMA (FP64 tensor core), DFMA, LDGSTS (cp.async), UTMALDG / UBLKCP (TMA), LDS / STS.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2503_17528_b200", "libserinv.so")
KEY = ["DMMA", "DFMA", "DMUL", "DADD", "MUFU", "LDGSTS", "UTMALDG", "UBLKCP", "LDS", "STS", "LDG", "STG", "SHFL",
       "BAR", "LDL", "STL", "ATOMG", "RED"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kern, hist = None, collections.defaultdict(collections.Counter)
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            kern = m.group(1)
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m and kern:
            hist[kern][m.group(1)] += 1
    print(f"SASS histogram of {os.path.relpath(LIB, ROOT)} (cuobjdump -sass; static instruction counts)")
    for k in sorted(hist):
        h = hist[k]
        print(f"\n== {k}: {sum(h.values())} instructions")
        print("  key: " + ", ".join(f"{op} {h.get(op, 0)}" for op in KEY))
        print("  top: " + ", ".join(f"{op} {c}" for op, c in h.most_common(14)))
    # the DMMA shape
    shapes = collections.Counter(re.findall(r"DMMA\.[0-9x]+", out))
    print("\nDMMA variants: " + ", ".join(f"{s} {c}" for s, c in shapes.items()))


if __name__ == "__main__":
    sys.exit(main())
