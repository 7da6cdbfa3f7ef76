"""Build libserinv.so (sm_100a) in-tree with nvcc.

    python -m paper_2503_17528_b200.build        # or __graft_entry__.build()

Flags: -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo; the host graph
builder (graph.cpp) is compiled by the same nvcc invocation as C++17.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libserinv.so")
SOURCES = ["exec.cu", "serinv.cu", "graph.cpp", "comm.cpp", "sb.cu"]
HEADERS = ["exec.h", "graph.h", "task.h", "dist_meta.h", "comm.h", "sb.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2", "-shared", "-ldl",
]


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "serinv.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = True) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [_nvcc()] + NVCC_FLAGS + ["-I" + os.path.join(ROOT, "include"), "-o", LIB + ".tmp"]
    cmd += [os.path.join(CSRC, f) for f in SOURCES]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_daginterp(verbose: bool = False) -> str:
    """Test tool (tools/libdaginterp.so): host interpreter of the task graphs."""
    out = os.path.join(ROOT, "tools", "libdaginterp.so")
    srcs = [os.path.join(ROOT, "tools", "daginterp.cpp"), os.path.join(CSRC, "graph.cpp")]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS]
    if os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out) for d in deps):
        return out
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", out + ".tmp"] + srcs
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv)
    build_daginterp(verbose=True)
