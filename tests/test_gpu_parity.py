"""GPU parity: libserinv (sm_100a) vs the CPU oracle, element by element per block.

Gate (north_star): relative Frobenius error <= 1e-10 per output block.
"""
import numpy as np
import pytest

import btagen
from oracle import invariants as inv, sequential as seq
from tests.gpu_util import to_dev, to_host, args

pytestmark = pytest.mark.gpu
TOL = 1e-10


def _sb():
    import paper_2503_17528_b200 as sb
    return sb


def _cmp(G, R, keys=("diag", "lower", "arrow", "tip"), tol=TOL):
    e, where = inv.max_block_err(G, R, keys)
    assert e <= tol, (e, where)
    return e


SHAPES = [(8, 4, 2), (3, 70, 5), (4, 130, 70), (5, 64, 0), (2, 200, 3), (1, 100, 10), (6, 5, 3),
          (7, 33, 1), (3, 128, 64), (2, 1, 1), (1, 1, 0), (9, 65, 65)]


@pytest.mark.parametrize("n,b,a", SHAPES)
@pytest.mark.parametrize("gen", ["g1", "g2"])
def test_selinv_small(n, b, a, gen):
    sb = _sb()
    A = btagen.generate(gen, 3, n, b, a)
    L, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.selinv(*args(D))
    _cmp(to_host(D), X)
    assert abs(ldg - ld) <= 1e-12 * max(1.0, abs(ld))


@pytest.mark.parametrize("n,b,a", SHAPES)
def test_pobtaf_then_pobtasi(n, b, a):
    sb = _sb()
    A = btagen.g2(5, n, b, a)
    L, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.pobtaf(*args(D))
    _cmp(to_host(D), L)
    assert abs(ldg - ld) <= 1e-12 * max(1.0, abs(ld))
    sb.pobtasi(*args(D))
    _cmp(to_host(D), X)


def test_pobtasi_from_oracle_factor():
    sb = _sb()
    A = btagen.g1(9, 6, 96, 7)
    L = seq.pobtaf(A)
    X = seq.pobtasi(L)
    D = to_dev(L)
    sb.pobtasi(*args(D))
    _cmp(to_host(D), X)


def test_c1_seeds():
    sb = _sb()
    for seed in range(1, 31):
        for gen in ("g1", "g2", "g2k"):
            A = btagen.generate(gen, seed, 8, 4, 2)
            L, X, ld = seq.selinv(A)
            D = to_dev(A)
            ldg = sb.selinv(*args(D))
            _cmp(to_host(D), X)
            assert abs(ldg - ld) <= 1e-12 * abs(ld)


@pytest.mark.parametrize("n,b,a,gen", [(32, 256, 16, "g2"), (16, 512, 64, "g1"), (12, 300, 20, "g2")])
def test_selinv_medium(n, b, a, gen):
    sb = _sb()
    A = btagen.generate(gen, 11, n, b, a)
    L, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.selinv(*args(D))
    _cmp(to_host(D), X)
    assert abs(ldg - ld) <= 1e-12 * abs(ld)


def test_deterministic_bits():
    import torch
    sb = _sb()
    A = btagen.g2(4, 10, 200, 9)
    outs = []
    for _ in range(3):
        D = to_dev(A)
        ld = sb.selinv(*args(D))
        torch.cuda.synchronize()
        outs.append((to_host(D), ld))
    for k in ("diag", "lower", "arrow", "tip"):
        assert np.array_equal(outs[0][0][k], outs[1][0][k]) and np.array_equal(outs[0][0][k], outs[2][0][k])
    assert outs[0][1] == outs[1][1] == outs[2][1]


def test_not_positive_definite_info():
    sb = _sb()
    A = btagen.g1(5, 5, 70, 3)
    A["diag"][2][10, 10] = -1e7
    with pytest.raises(seq.NotPositiveDefinite) as ei:
        seq.pobtaf(A)
    D = to_dev(A)
    with pytest.raises(sb.NotPositiveDefinite) as eg:
        sb.pobtaf(*args(D))
    assert eg.value.row == ei.value.row == 2 * 70 + 11


def test_not_positive_definite_tip():
    sb = _sb()
    A = btagen.g1(5, 3, 16, 4)
    A["tip"][2, 2] = -1e9
    D = to_dev(A)
    with pytest.raises(sb.NotPositiveDefinite) as eg:
        sb.selinv(*args(D))
    assert eg.value.row == 3 * 16 + 3


def test_launch_count_is_one_kernel():
    sb = _sb()
    A = btagen.g1(1, 4, 64, 4)
    D = to_dev(A)
    h = sb.default_handle()
    sb.selinv(*args(D), handle=h)
    assert h.last_launches() == 1


@pytest.mark.parametrize("n,b,a", [(9, 128, 8), (40, 64, 4), (5, 200, 0), (1, 64, 3), (10, 1024, 16)])
def test_selinv_host_streaming(n, b, a):
    """serinv_selinv_host: H2D / D2H stream with the computation (arrival / final counters)."""
    import torch
    sb = _sb()
    A = btagen.g2(6, n, b, a)
    L, X, ld = seq.selinv(A)
    host = {k: torch.from_numpy(np.ascontiguousarray(A[k])).pin_memory() for k in ("diag", "lower", "arrow", "tip")}
    out = {k: torch.empty_like(v).pin_memory() for k, v in host.items()}
    D = {k: torch.empty(v.shape, dtype=torch.float64, device="cuda") for k, v in host.items()}
    for rep in range(2):
        ldg = sb.selinv_host(host, D, out)
        G = {k: v.numpy() for k, v in out.items()}
        e, where = inv.max_block_err(G, X)
        assert e <= TOL, (e, where)
        assert abs(ldg - ld) <= 1e-12 * max(1.0, abs(ld))


@pytest.mark.parametrize("opt", ["carry_min_b=64", "carry_min_b=64,twist_min_n=0", "chol8=0", "early_sig=0",
                                 "wide_min_wave=1", "fuse_trsm=1,split_chain=0", "chain_step=1"])
def test_scheduling_variants_parity(opt, monkeypatch):
    """Graph-build options (SERINV_OPT, read when a handle builds a graph) change the
    task structure -- carried chain, one-sided order, 16x16-leaf POTRF, late
    publication, wide tasks, fused TRSM -- never the results."""
    sb = _sb()
    monkeypatch.setenv("SERINV_OPT", opt)
    h = sb.Handle(0)
    A = btagen.g2(31, 6, 192, 5)
    L, X, ld = seq.selinv(A)
    D = to_dev(A)
    ldg = sb.selinv(*args(D), handle=h)
    assert inv.max_block_err(to_host(D), X)[0] <= TOL
    assert abs(ldg - ld) <= 1e-12 * abs(ld)
    D = to_dev(A)
    sb.pselinv(*args(D), 3, handle=h)
    assert inv.max_block_err(to_host(D), X)[0] <= TOL
