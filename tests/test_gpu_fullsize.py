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


@pytest.mark.parametrize("cfg", [(256, 512, 16, "g2")])   # C2 / C4 on G1 seed 0: test_gpu_timed_inputs.py
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


def _distributed_closed_form_check(n_loc, b, a, P, samples, tol=1e-10):
    """bench.py --gpus P's launch configuration (plan_ends with auto_r, Q = dist_auto_q,
    ppobtaf_q -> all-gather -> ppobtasi_q per rank), the P ranks simulated one after the
    other on one B200, against the G2K closed form on sampled global blocks."""
    import torch
    sb = _sb()
    from paper_2503_17528_b200 import distributed as sd
    n = n_loc * P
    A, fac = btagen.g2k(2, n, b, a, with_factors=True)
    c = cf.closed_form(n, b, a, fac)
    parts = sb.plan_ends(n, P, sd.auto_r(b))
    Q = sd.dist_auto_q(min(e - s for s, e in parts), b)
    h = sb.default_handle()
    ranks = []
    for p, (s, e) in enumerate(parts):
        loc = sd.local_blocks(A, s, e, last=(p == P - 1))
        D = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in loc.items()}
        ranks.append((s, e, D, sd.DistContext(h, P, p, n, s, e - s, b, a, Q=Q)))
    for s, e, D, ctx in ranks:
        sd.ppobtaf(ctx, D)
    recv = torch.cat([ctx.send for _, _, _, ctx in ranks])
    for s, e, D, ctx in ranks:
        ctx.recv.copy_(recv)
        sd.ppobtasi(ctx, D)
    torch.cuda.synchronize()
    for s, e, D, ctx in ranks:
        assert int(ctx.info.item()) == 0
        assert abs(float(ctx.logdet.item()) - c.logdet()) <= 1e-11 * abs(c.logdet())
        for i in [i for i in samples if s <= i < e]:
            assert inv.rel_err(D["diag"][i - s].cpu().numpy(), c.X_block(i, i)) <= tol, ("diag", i)
            if i + 1 < n:
                assert inv.rel_err(D["lower"][i - s].cpu().numpy(), c.X_block(i + 1, i)) <= tol, ("lower", i)
            if a:
                assert inv.rel_err(D["arrow"][i - s].cpu().numpy(), c.X_arrow(i)) <= tol, ("arrow", i)
        if a:
            assert inv.rel_err(D["tip"].cpu().numpy(), c.X_tip()) <= tol
    del ranks
    torch.cuda.empty_cache()


def test_c4_distributed_closed_form_p4():
    # C4 weak scaling at P = 4 (n = 256 per rank, Q = 4 sub-partitions, nested reduced solve)
    n = 1024
    _distributed_closed_form_check(256, 512, 16, 4, [0, 1, 63, 64, 255, 256, 511, 512, 767, 768, n - 2, n - 1])


def test_c5_distributed_closed_form_p2():
    # C5 at P = 2 (n = 16384 per rank, Q = 256, reduced system of 1022 blocks nested)
    n = 32768
    _distributed_closed_form_check(16384, 64, 8, 2, [0, 1, 63, 64, 8191, 16383, 16384, 16385, 24000, n - 2, n - 1])
