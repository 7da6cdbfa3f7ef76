"""Distributed PPOBTAF / PPOBTASI (one process per GPU; Alg. 3-6).

Filled in by the distributed milestone; see include/serinv.h."""
from __future__ import annotations


def ppobtaf(*args, **kwargs):  # pragma: no cover - replaced by the distributed milestone
    raise NotImplementedError("ppobtaf: distributed path not built yet")


def ppobtasi(*args, **kwargs):  # pragma: no cover
    raise NotImplementedError("ppobtasi: distributed path not built yet")
