"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (serinv_selinv, one persistent launch):

* C2 (n=128, b=1024, a=64) and C4 (n=256, b=512, a=16): element-by-element
  against the oracle (numpy/scipy FP64 finishes in seconds on the host).
* C3 (n=365, b=2048, a=4) and C5 (n=16384, b=64, a=8): the G2K family's
  closed-form selected inverse on sampled blocks (oracle/closed_form.py) plus
  the size-independent invariant (X A)|pattern = I on sampled blocks.
"""
import numpy as np
import pytest

import btagen
from oracle import closed_form as cf, invariants as inv, sequential as seq
from tests.gpu_util import args, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _sb():
    import paper_2503_17528_b200 as sb
    return sb


@pytest.mark.parametrize("cfg", [(128, 1024, 64, "g1"), (256, 512, 16, "g2")])
def test_full_size_against_oracle(cfg):
    n, b, a, gen = cfg
    sb = _sb()
    A = btagen.generate(gen, 1, n, b, a)
    L, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.selinv(*args(D))
    G = to_host(D)
    e, where = inv.max_block_err(G, X)
    assert e <= TOL, (e, where)
    assert abs(ldg - ld) <= 1e-12 * abs(ld)


def _closed_form_check(n, b, a, samples, tol=1e-10, Ps=None):
    import torch
    sb = _sb()
    A, fac = btagen.g2k(2, n, b, a, with_factors=True)
    c = cf.closed_form(n, b, a, fac)
    D = to_dev(A)
    ldg = sb.selinv(*args(D)) if Ps is None else sb.pselinv(*args(D), Ps)
    assert abs(ldg - c.logdet()) <= 1e-11 * abs(c.logdet())
    for i in samples:
        Xd = D["diag"][i].cpu().numpy()
        assert inv.rel_err(Xd, c.X_block(i, i)) <= tol, ("diag", i)
        if i + 1 < n:
            assert inv.rel_err(D["lower"][i].cpu().numpy(), c.X_block(i + 1, i)) <= tol, ("lower", i)
        if a:
            assert inv.rel_err(D["arrow"][i].cpu().numpy(), c.X_arrow(i)) <= tol, ("arrow", i)
    if a:
        assert inv.rel_err(D["tip"].cpu().numpy(), c.X_tip()) <= tol
    del D
    torch.cuda.empty_cache()


def test_c5_closed_form():
    n = 16384
    _closed_form_check(n, 64, 8, [0, 1, 2, 777, 8191, n // 2 + 3, n - 2, n - 1])


def test_c5_closed_form_nested_auto_plan():
    # the launch configuration bench.py times for small b: the library's nested plan
    n = 16384
    Ps = _sb().auto_partitions(n, 64)
    assert len(Ps) >= 2
    _closed_form_check(n, 64, 8, [0, 1, 2, 127, 128, 777, 8191, n // 2 + 3, n - 2, n - 1], Ps=Ps)


@pytest.mark.slow
def test_c3_closed_form():
    n = 365
    _closed_form_check(n, 2048, 4, [0, 1, 180, n - 2, n - 1])
