"""Helpers for the -m gpu parity tests (host <-> device marshalling only)."""
import numpy as np

KEYS = ("diag", "lower", "arrow", "tip")


def to_dev(A):
    import torch
    out = {}
    for k in KEYS:
        out[k] = torch.from_numpy(np.ascontiguousarray(A[k])).to("cuda")
    return out


def to_host(D):
    return {k: D[k].cpu().numpy() for k in KEYS}


def args(D):
    n = D["diag"].shape[0]
    a = D["tip"].shape[0]
    return (D["diag"], D["lower"] if n > 1 else None, D["arrow"] if a > 0 else None, D["tip"] if a > 0 else None)
