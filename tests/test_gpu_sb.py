"""GPU parity of the small-block engine (serinv_sb_selinv, b <= 64, a <= 16) against
the CPU oracle: the partitioned method with nested solving (Sec. 3, Alg. 3-6,
Sec. 4.2) gives X = A^{-1} on the pattern and log det A for every plan.

Shapes span padded blocks (b < 64), a = 0 / 1 / odd / 16, one-chain plans, single
and multi-level nesting, two-block middle partitions and one-block end partitions;
full size: BASELINE C5 (n=16384, b=64, a=8) in the bench's launch configuration
(the library's plan) on G2K (closed form) and on the bench input G1 seed 0
(oracle on a prefix-free property: sampled (XA)|pattern = I).
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


CASES = [
    # (n, b, a, Ps)
    (1, 64, 8, []), (2, 64, 8, []), (7, 64, 8, []), (5, 64, 0, []), (6, 13, 3, []), (4, 1, 1, []),
    (8, 64, 8, [2]), (9, 64, 8, [3]), (12, 64, 16, [4]), (10, 32, 5, [4]), (11, 64, 1, [5]),
    (3, 64, 8, [2]), (5, 40, 0, [3]), (40, 64, 8, [5, 3]), (60, 64, 8, [10, 4]), (64, 24, 7, [8, 4, 2]),
    (97, 64, 8, [12, 5, 3]), (30, 64, 16, [14]), (33, 17, 9, [6, 3]),
]


@pytest.mark.parametrize("n,b,a,Ps", CASES)
@pytest.mark.parametrize("gen", ["g1", "g2"])
def test_sb_against_oracle(n, b, a, Ps, gen):
    sb = _sb()
    A = btagen.generate(gen, 4, n, b, a)
    _, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.selinv_sb(*args(D), Ps)
    e, where = inv.max_block_err(to_host(D), X)
    assert e <= TOL, (e, where)
    assert abs(ldg - ld) <= 1e-12 * max(1.0, abs(ld))


def test_sb_auto_plan_mid_size():
    # the library's plan (nested) on n = 3000 blocks: every partition kind, two levels
    sb = _sb()
    n, b, a = 3000, 64, 8
    Ps = sb.sb_auto_plan(n, b, a)
    assert len(Ps) >= 2
    A = btagen.g2(6, n, b, a)
    _, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.selinv_sb(*args(D))
    e, where = inv.max_block_err(to_host(D), X)
    assert e <= TOL, (e, where)
    assert abs(ldg - ld) <= 1e-12 * abs(ld)


def test_sb_deterministic():
    sb = _sb()
    A = btagen.g1(8, 200, 64, 8)
    outs = []
    for _ in range(2):
        D = to_dev(A)
        ld = sb.selinv_sb(*args(D), [20, 6])
        outs.append((to_host(D), ld))
    for k in ("diag", "lower", "arrow", "tip"):
        assert np.array_equal(outs[0][0][k], outs[1][0][k]), k
    assert outs[0][1] == outs[1][1]


@pytest.mark.parametrize("blk,row", [(0, 5), (37, 0), (63, 63), ("tip", 2)])
def test_sb_not_positive_definite(blk, row):
    # dpotrf semantics: the 1-based global row of the first non-positive pivot, log det NaN
    sb = _sb()
    n, b, a = 64, 64, 8
    A = btagen.g1(3, n, b, a)
    if blk == "tip":
        A["tip"][row, row] = -1e6
        want = n * b + row + 1
    else:
        A["diag"][blk][row, row] = -1e6
        want = blk * b + row + 1
    D = to_dev(A)
    with pytest.raises(sb.NotPositiveDefinite) as ei:
        sb.selinv_sb(*args(D), [8, 4])
    assert ei.value.row == want


def test_sb_launch_count():
    sb = _sb()
    A = btagen.g1(1, 40, 64, 8)
    D = to_dev(A)
    h = sb.default_handle()
    sb.selinv_sb(*args(D), [5, 3], handle=h)
    # factor + inverse kernel per level (2 nested + the last chain), plus the level-0
    # W-form precompute on the side stream (sb_pre_kernel)
    assert h.last_launches() == 2 * 3 + 1


def test_sb_rejects_unsupported_shapes():
    import ctypes
    from paper_2503_17528_b200 import _lib
    L = _lib.lib()
    nb = ctypes.c_size_t(0)
    arr = (ctypes.c_int * 1)(2)
    assert L.serinv_sb_ws(10, 65, 4, 0, arr, ctypes.byref(nb)) == 1005  # b > 64
    assert L.serinv_sb_ws(10, 64, 17, 0, arr, ctypes.byref(nb)) == 1005  # a > 16
    bad = (ctypes.c_int * 1)(9)
    assert L.serinv_sb_ws(10, 64, 4, 1, bad, ctypes.byref(nb)) == 1007    # 9 partitions of 10 blocks


# ----------------------------------------------------------------------------- C5 full size
C5 = (16384, 64, 8)
C5_SAMPLES = [0, 1, 2, 3, 110, 111, 112, 777, 4095, 8191, 8192, 12000, 16270, 16381, 16382, 16383]


def test_c5_sb_closed_form():
    import torch
    sb = _sb()
    n, b, a = C5
    A, fac = btagen.g2k(2, n, b, a, with_factors=True)
    c = cf.closed_form(n, b, a, fac)
    D = to_dev(A)
    ldg = sb.selinv_sb(*args(D))
    assert abs(ldg - c.logdet()) <= 1e-11 * abs(c.logdet())
    for i in C5_SAMPLES:
        assert inv.rel_err(D["diag"][i].cpu().numpy(), c.X_block(i, i)) <= TOL, ("diag", i)
        if i + 1 < n:
            assert inv.rel_err(D["lower"][i].cpu().numpy(), c.X_block(i + 1, i)) <= TOL, ("lower", i)
        assert inv.rel_err(D["arrow"][i].cpu().numpy(), c.X_arrow(i)) <= TOL, ("arrow", i)
    assert inv.rel_err(D["tip"].cpu().numpy(), c.X_tip()) <= TOL
    del D
    torch.cuda.empty_cache()


def test_c5_sb_bench_input_residual_and_logdet():
    # the bench's own input (G1 seed 0) in the bench's launch configuration: sampled
    # (XA)|pattern = I (sensitivity-pinned residual) and log det against the executor path
    import torch
    from tests.test_gpu_timed_inputs import XA_TOL, _xa_sampled
    sb = _sb()
    n, b, a = C5
    A = btagen.g1_torch(0, n, b, a, device="cuda")
    X = {k: v.clone() for k, v in A.items()}
    ld = sb.selinv_sb(*args(X))
    res = _xa_sampled(X, A, C5_SAMPLES)
    assert res <= XA_TOL, res
    Y = {k: v.clone() for k, v in A.items()}
    ld2 = sb.selinv(*args(Y))
    assert abs(ld - ld2) <= 1e-12 * abs(ld2)
    for k in ("diag", "lower", "arrow", "tip"):
        d = float((X[k] - Y[k]).norm() / Y[k].norm())
        assert d <= 1e-12, (k, d)
    X["diag"][8191][7, 9] += 1e-8 * float(X["diag"].abs().max())
    assert _xa_sampled(X, A, [8191]) >= 1e-9
    del A, X, Y
    torch.cuda.empty_cache()
