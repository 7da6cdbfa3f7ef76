"""GPU parity of the partitioned method (Sec. 3, Alg. 3-6) against the oracle.

* serinv_pselinv: all partitions + reduced system in one graph on one device.
* serinv_ppobtaf / serinv_ppobtasi: the per-rank distributed entry points, with
  P ranks simulated on one GPU (the all-gather replaced by a device copy of the
  records in rank order -- exactly the buffer NCCL would produce).
"""
import ctypes

import numpy as np
import pytest

import btagen
from oracle import invariants as inv, parallel as par, sequential as seq
from tests.gpu_util import args, to_dev, to_host

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _sb():
    import paper_2503_17528_b200 as sb
    return sb


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("n,b,a,gen", [(17, 64, 4, "g2"), (24, 70, 5, "g2"), (30, 33, 0, "g1"), (16, 128, 16, "g1")])
def test_pselinv(P, n, b, a, gen):
    if n < 2 * P - 1:
        pytest.skip("too few blocks")
    sb = _sb()
    A = btagen.generate(gen, 13 + P, n, b, a)
    L, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.pselinv(*args(D), P)
    e, where = inv.max_block_err(to_host(D), X)
    assert e <= TOL, (e, where)
    assert abs(ldg - ld) <= 1e-12 * max(1.0, abs(ld))


@pytest.mark.parametrize("Ps", [[4, 2], [8, 4], [16, 5, 2], [6, 3]])
@pytest.mark.parametrize("n,b,a,gen", [(48, 64, 4, "g2"), (40, 70, 5, "g2"), (64, 33, 0, "g1")])
def test_pselinv_nested(Ps, n, b, a, gen):
    # nested solving (Sec. 4.2): same X and log det as the sequential oracle
    sb = _sb()
    A = btagen.generate(gen, 7 + len(Ps), n, b, a)
    L, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.pselinv(*args(D), Ps)
    e, where = inv.max_block_err(to_host(D), X)
    assert e <= TOL, (Ps, e, where)
    assert abs(ldg - ld) <= 1e-12 * max(1.0, abs(ld))


def test_pselinv_nested_not_positive_definite():
    sb = _sb()
    n, b, a = 40, 16, 2
    A = btagen.g1(5, n, b, a)
    blk = par.plan(n, 4, 1.0)[1][0]  # a level-0 boundary block, eliminated at level 1
    A["diag"][blk][2, 2] = -1e6
    D = to_dev(A)
    with pytest.raises(sb.NotPositiveDefinite) as ei:
        sb.pselinv(*args(D), [4, 2])
    assert ei.value.row == blk * b + 3


def test_pselinv_ratio_and_smallest_middles():
    sb = _sb()
    A = btagen.g2(3, 9, 48, 3)
    L, X, ld = seq.selinv(A)
    for r in (0.1, 1.0, 1.8, 2.25):
        D = to_dev(A)
        sb.pselinv(*args(D), 4, r)
        assert inv.max_block_err(to_host(D), X)[0] <= TOL


def _run_distributed_on_one_gpu(A, P, r=1.0, Q=1):
    """Simulate P ranks of serinv_ppobtaf / all-gather / serinv_ppobtasi on cuda:0."""
    import torch
    sb = _sb()
    from paper_2503_17528_b200 import distributed as sd
    n, b = A["diag"].shape[0], A["diag"].shape[1]
    a = A["tip"].shape[0]
    parts = sb.plan(n, P, r)
    h = sb.default_handle()
    ranks = []
    for p, (s, e) in enumerate(parts):
        loc = sd.local_blocks(A, s, e, last=(p == P - 1))
        D = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in loc.items()}
        ctx = sd.DistContext(h, P, p, n, s, e - s, b, a, Q=Q)
        ranks.append((s, e, D, ctx))
    for s, e, D, ctx in ranks:
        sd.ppobtaf(ctx, D)
    recv = torch.cat([ctx.send for _, _, _, ctx in ranks])
    lds = []
    for s, e, D, ctx in ranks:
        ctx.recv.copy_(recv)
        sd.ppobtasi(ctx, D)
    torch.cuda.synchronize()
    for s, e, D, ctx in ranks:
        assert int(ctx.info.item()) == 0
        lds.append(float(ctx.logdet.item()))
    return ranks, lds


@pytest.mark.parametrize("P", [1, 2, 3, 4])
@pytest.mark.parametrize("n,b,a", [(12, 64, 4), (15, 70, 0), (20, 40, 7)])
def test_distributed_entry_points(P, n, b, a):
    A = btagen.g2(21, n, b, a)
    L, X, ld = seq.selinv(A)
    ranks, lds = _run_distributed_on_one_gpu(A, P)
    assert len(set(lds)) == 1                    # bit-identical on every rank
    assert abs(lds[0] - ld) <= 1e-12 * abs(ld)
    for s, e, D, ctx in ranks:
        G = {k: v.cpu().numpy() for k, v in D.items()}
        for i in range(s, e):
            assert inv.rel_err(G["diag"][i - s], X["diag"][i]) <= TOL
            if a:
                assert inv.rel_err(G["arrow"][i - s], X["arrow"][i]) <= TOL
            if i < n - 1:
                assert inv.rel_err(G["lower"][i - s], X["lower"][i]) <= TOL
        if a:
            assert inv.rel_err(G["tip"], X["tip"]) <= TOL


@pytest.mark.parametrize("P,Q", [(1, 3), (2, 2), (3, 4), (2, 40)])
@pytest.mark.parametrize("n,b,a", [(170, 64, 4), (175, 70, 0)])
def test_distributed_subpartitions(P, Q, n, b, a):
    # serinv_ppobtaf_q / serinv_ppobtasi_q: Q sub-partitions per rank; (2, 40) has a
    # reduced system of 158 blocks, solved by the nested algorithm
    A = btagen.g2(23, n, b, a)
    L, X, ld = seq.selinv(A)
    ranks, lds = _run_distributed_on_one_gpu(A, P, Q=Q)
    assert len(set(lds)) == 1
    assert abs(lds[0] - ld) <= 1e-12 * abs(ld)
    for s, e, D, ctx in ranks:
        G = {k: v.cpu().numpy() for k, v in D.items()}
        for i in range(s, e):
            assert inv.rel_err(G["diag"][i - s], X["diag"][i]) <= TOL
            if a:
                assert inv.rel_err(G["arrow"][i - s], X["arrow"][i]) <= TOL
            if i < n - 1:
                assert inv.rel_err(G["lower"][i - s], X["lower"][i]) <= TOL
        if a:
            assert inv.rel_err(G["tip"], X["tip"]) <= TOL


def test_partitioned_factor_blocks_match_oracle_permuted_factor():
    """The eliminated blocks after the partitioned run's factor phase equal the
    oracle's PERMUTED_POBTAF factor (same algorithm, Alg. 4) for a middle partition."""
    sb = _sb()
    import torch
    from paper_2503_17528_b200 import distributed as sd
    A = btagen.g2(8, 14, 32, 3)
    R = par.pselinv(A, 3)
    s, e = sb.plan(14, 3, 1.0)[1]
    loc = sd.local_blocks(A, s, e, last=False)
    D = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in loc.items()}
    ctx = sd.DistContext(sb.default_handle(), 3, 1, 14, s, e - s, 32, 3)
    sd.ppobtaf(ctx, D)
    torch.cuda.synchronize()
    G = {k: v.cpu().numpy() for k, v in D.items()}
    for i in range(s + 1, e - 1):   # interior blocks of the middle partition: factor L
        assert inv.rel_err(G["diag"][i - s], R["L"]["diag"][i]) <= TOL
        assert inv.rel_err(G["arrow"][i - s], R["L"]["arrow"][i]) <= TOL


def test_twisted_last_partition_factor_is_reversed_pobtaf():
    """Reading R14: the last partition eliminates blocks e-1, ..., s+1 bottom-up, i.e.
    Alg. 1 on the block-reversed BTA matrix (again BTA); its diagonal and arrow factor
    blocks equal the oracle's POBTAF of the reversed matrix."""
    sb = _sb()
    import torch
    from paper_2503_17528_b200 import distributed as sd
    n, b, a, P = 14, 32, 3, 3
    A = btagen.g2(9, n, b, a)
    s, e = sb.plan(n, P, 1.0)[P - 1]
    assert e == n
    # block-reversed matrix of blocks e-1 .. s (plus the tip): lower_rev[k] = A_{j-1,j} = lower[j-1]^T
    blocks = list(range(e - 1, s - 1, -1))
    Rv = {"diag": np.stack([A["diag"][j] for j in blocks]),
          "lower": np.stack([A["lower"][j - 1].T for j in blocks[:-1]]),
          "arrow": np.stack([A["arrow"][j] for j in blocks]),
          "tip": np.zeros((a, a))}
    loc = sd.local_blocks(A, s, e, last=True)
    D = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in loc.items()}
    ctx = sd.DistContext(sb.default_handle(), P, P - 1, n, s, e - s, b, a)
    sd.ppobtaf(ctx, D)
    torch.cuda.synchronize()
    G = {k: v.cpu().numpy() for k, v in D.items()}
    # the factor of the reversed chain: L_kk = chol(...) in the same elimination order
    import scipy.linalg as sla
    Dw = {k: v.copy() for k, v in Rv.items()}
    for k in range(len(blocks) - 1):   # Alg. 1 l.2-6 on the reversed matrix (no tip needed)
        Lkk = np.linalg.cholesky(Dw["diag"][k])
        Lnext = sla.solve_triangular(Lkk, Dw["lower"][k].T, lower=True).T
        Larr = sla.solve_triangular(Lkk, Dw["arrow"][k].T, lower=True).T
        Dw["diag"][k + 1] -= Lnext @ Lnext.T
        Dw["arrow"][k + 1] -= Larr @ Lnext.T
        j = blocks[k]
        assert inv.rel_err(np.tril(G["diag"][j - s]), Lkk) <= TOL
        assert inv.rel_err(G["arrow"][j - s], Larr) <= TOL
