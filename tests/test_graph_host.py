"""Host logic of the product: the task-graph builder and scheduler (graph.cpp),
checked on CPU by executing the emitted task lists with the host interpreter
test tool (tools/daginterp.cpp, plain loops).  The interpreter also asserts
that every wait is satisfied at claim time, i.e. that the emission order is a
valid topological order (the persistent executor's deadlock-freedom premise).

This validates dependencies, block/tile locations, fusion and the partitioned
assembly; the CUDA tile kernels themselves are covered by the -m gpu tests.
"""
import ctypes

import numpy as np
import pytest

import btagen
from oracle import invariants as inv, parallel as par, sequential as seq

_lib = None


def lib():
    global _lib
    if _lib is None:
        from paper_2503_17528_b200.build import build_daginterp
        _lib = ctypes.CDLL(build_daginterp())
    return _lib


P_ = ctypes.c_void_p
KEYS = ("diag", "lower", "arrow", "tip")


def prep(A):
    A = {k: np.ascontiguousarray(np.array(A[k], dtype=np.float64)) for k in KEYS}
    n, b, a = A["diag"].shape[0], A["diag"].shape[1], A["tip"].shape[0]
    if A["lower"].size == 0:
        A["lower"] = np.zeros((1, b, b))
    if A["arrow"].size == 0:
        A["arrow"] = np.zeros((1, 1, b))
    if A["tip"].size == 0:
        A["tip"] = np.zeros((1, 1))
    return A, n, b, a


def cut(R, X):
    a = X["tip"].shape[0]
    return {k: (R[k][:X[k].shape[0]] if k != "tip" else R[k][:a, :a]) for k in X}


def ptrs(A):
    return [A[k].ctypes.data_as(P_) for k in KEYS]


def run_seq(kind, A0, grid=16, ug=4, si_split=-1):
    A, n, b, a = prep(A0)
    ld, info, nt = ctypes.c_double(0), ctypes.c_int(0), ctypes.c_int64(0)
    rc = lib().dag_run_sequential(kind, ctypes.c_int64(n), ctypes.c_int64(b), ctypes.c_int64(a), *ptrs(A),
                                  ctypes.byref(ld), ctypes.byref(info), grid, ug, ctypes.byref(nt), si_split)
    assert rc == 0
    return A, ld.value, info.value


SHAPES = [(8, 4, 2), (3, 70, 5), (4, 130, 70), (5, 64, 0), (2, 200, 3), (1, 100, 10), (6, 5, 3), (1, 1, 0),
          (3, 129, 1)]


@pytest.mark.parametrize("n,b,a", SHAPES)
def test_sequential_graphs(n, b, a):
    A0 = btagen.g2(1, n, b, a)
    L, X, ld = seq.selinv(A0)
    R, ldr, info = run_seq(2, A0)
    assert info == 0
    assert inv.max_block_err(cut(R, X), X)[0] < 1e-12
    assert abs(ldr - ld) <= 1e-12 * max(1, abs(ld))
    F, ldf, info = run_seq(0, A0)
    assert inv.max_block_err(cut(F, L), L)[0] < 1e-12
    assert abs(ldf - ld) <= 1e-12 * max(1, abs(ld))
    S, _, info = run_seq(1, L)
    assert inv.max_block_err(cut(S, X), X)[0] < 1e-12


@pytest.mark.parametrize("n,b,a", [(6, 70, 5), (3, 64, 0), (1, 30, 2)])
def test_streaming_io_graph(n, b, a):
    # kind 6 (serinv_selinv_host): same results as selinv, all final-X counters complete
    A0 = btagen.g2(2, n, b, a)
    L, X, ld = seq.selinv(A0)
    R, ldr, info = run_seq(6, A0)
    assert info == 0
    assert inv.max_block_err(cut(R, X), X)[0] < 1e-12
    assert abs(ldr - ld) <= 1e-12 * max(1, abs(ld))


@pytest.mark.parametrize("ug", [1, 2, 7])
@pytest.mark.parametrize("grid", [1, 3, 296])
def test_schedule_options_do_not_change_results(ug, grid):
    A0 = btagen.g1(4, 4, 150, 9)
    L, X, ld = seq.selinv(A0)
    R, ldr, info = run_seq(2, A0, grid=grid, ug=ug)
    assert inv.max_block_err(cut(R, X), X)[0] < 1e-12


@pytest.mark.parametrize("si_split", [0, 16, 64, 100])
def test_split_k_inversion(si_split):
    # the Takahashi tile tasks split along K into partial GEMMs + fixed-order REDUCE
    A0 = btagen.g2(3, 5, 130, 20)
    L, X, ld = seq.selinv(A0)
    for kind, src, ref in ((2, A0, X), (1, L, X)):
        R, _, info = run_seq(kind, src, si_split=si_split)
        assert info == 0
        assert inv.max_block_err(cut(R, ref), ref)[0] < 1e-12


def test_info_first_bad_pivot():
    A0 = btagen.g1(5, 5, 70, 3)
    A0["diag"][2][10, 10] = -1e7
    _, ld, info = run_seq(0, A0)
    assert info == 2 * 70 + 11
    assert np.isnan(ld)


@pytest.mark.parametrize("twist_last", [1, 0])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("n,b,a", [(17, 4, 2), (24, 70, 5), (30, 8, 0), (16, 65, 3)])
def test_pselinv_and_distributed_graphs(P, n, b, a, twist_last, monkeypatch):
    # twist_last=1: the last partition eliminates bottom-up (reading R14), the
    # reduced system has 2P-2 blocks; 0: the paper's scheme (2P-1)
    monkeypatch.setenv("SERINV_OPT", f"twist_last={twist_last}")
    if n < 2 * P - 1:
        pytest.skip("too few blocks")
    A0 = btagen.g2(7, n, b, a)
    L, X, ld = seq.selinv(A0)
    for runner in ("dag_run_pselinv", "dag_run_distributed"):
        A, n_, b_, a_ = prep(A0)
        ldv, info = ctypes.c_double(0), ctypes.c_int(0)
        if runner == "dag_run_pselinv":
            nt = ctypes.c_int64(0)
            rc = lib().dag_run_pselinv(ctypes.c_int64(n), ctypes.c_int64(b), ctypes.c_int64(a), P,
                                       ctypes.c_double(1.0), *ptrs(A), ctypes.byref(ldv), ctypes.byref(info), 16,
                                       ctypes.byref(nt))
        else:
            rc = lib().dag_run_distributed(ctypes.c_int64(n), ctypes.c_int64(b), ctypes.c_int64(a), P,
                                           ctypes.c_double(1.0), *ptrs(A), ctypes.byref(ldv), ctypes.byref(info))
        assert rc == 0 and info.value == 0
        e, where = inv.max_block_err(cut(A, X), X)
        assert e < 1e-11, (runner, e, where)
        assert abs(ldv.value - ld) <= 1e-12 * max(1, abs(ld))


@pytest.mark.parametrize("n,b,a,P,Q", [(24, 4, 2, 2, 2), (40, 8, 3, 3, 3), (30, 5, 0, 1, 4), (33, 6, 2, 2, 5),
                                       (80, 4, 2, 4, 10), (140, 3, 1, 2, 35)])
@pytest.mark.parametrize("dist_len", [0, 6])
def test_distributed_subpartitions(n, b, a, P, Q, dist_len, monkeypatch):
    # each rank splits its blocks into Q sub-partitions (serinv_ppobtaf_q / _q); the
    # last two cases (and dist_len = 6: partitions of ~6 blocks) nest the reduced solve
    monkeypatch.setenv("SERINV_OPT", f"dist_len={dist_len}")
    A0 = btagen.g2(7, n, b, a)
    L, X, ld = seq.selinv(A0)
    A, n_, b_, a_ = prep(A0)
    ldv, info = ctypes.c_double(0), ctypes.c_int(0)
    rc = lib().dag_run_distributed_q(ctypes.c_int64(n), ctypes.c_int64(b), ctypes.c_int64(a), P, Q,
                                     ctypes.c_double(1.0), *ptrs(A), ctypes.byref(ldv), ctypes.byref(info))
    assert rc == 0 and info.value == 0
    e, where = inv.max_block_err(cut(A, X), X)
    assert e < 1e-11, (e, where)
    assert abs(ldv.value - ld) <= 1e-12 * max(1, abs(ld))


def test_partition_plan_matches_oracle_reading():
    import paper_2503_17528_b200._lib  # noqa: F401  (the product plan lives in libserinv)
    # serinv_plan is exported by libserinv.so; compare with the oracle's reading R6 when available
    try:
        from paper_2503_17528_b200 import plan
        for n in range(1, 40):
            for P in range(1, 7):
                for r in (0.5, 1.0, 1.8, 2.25):
                    if n < 2 * P - 1:
                        continue
                    assert plan(n, P, r) == par.plan(n, P, r)
    except ImportError:
        pytest.skip("libserinv.so not built")


def run_nested(A0, Ps, r=1.0, grid=16):
    A, n, b, a = prep(A0)
    ldv, info, nt = ctypes.c_double(0), ctypes.c_int(0), ctypes.c_int64(0)
    arr = (ctypes.c_int * len(Ps))(*Ps)
    rc = lib().dag_run_pselinv_nested(ctypes.c_int64(n), ctypes.c_int64(b), ctypes.c_int64(a), len(Ps), arr,
                                      ctypes.c_double(r), *ptrs(A), ctypes.byref(ldv), ctypes.byref(info), grid,
                                      ctypes.byref(nt))
    return rc, A, ldv.value, info.value


@pytest.mark.parametrize("Ps", [[4, 2], [5, 3], [8, 3], [8, 4, 2], [3, 2]])
@pytest.mark.parametrize("n,b,a", [(40, 4, 2), (33, 9, 0), (48, 66, 3)])
def test_nested_pselinv_graphs(Ps, n, b, a):
    # nested solving (Sec. 4.2): the reduced system of level k is itself solved by
    # the partitioned algorithm with Ps[k+1] partitions; X and log det must equal
    # the sequential selected inversion for any nesting (SURVEY 8(c) O3 pin)
    A0 = btagen.g2(11, n, b, a)
    L, X, ld = seq.selinv(A0)
    rc, R, ldv, info = run_nested(A0, Ps)
    assert rc == 0 and info == 0
    e, where = inv.max_block_err(cut(R, X), X)
    assert e < 1e-11, (Ps, e, where)
    assert abs(ldv - ld) <= 1e-12 * max(1, abs(ld))


def test_nested_info_reports_global_row():
    # a bad pivot inside a block that is eliminated at nesting level 1 (a partition
    # boundary of level 0) is reported with its global row
    n, b, a = 40, 6, 2
    A0 = btagen.g1(5, n, b, a)
    starts = par.plan(n, 4, 1.0)
    blk = starts[1][0]  # first block of partition 1: a level-0 boundary
    A0["diag"][blk][2, 2] = -1e6
    rc, R, ldv, info = run_nested(A0, [4, 2])
    assert rc == 0
    assert info == blk * b + 3
    assert np.isnan(ldv)


def test_auto_partitions_policy():
    out = (ctypes.c_int * 8)()
    k = lib().dag_auto_partitions(ctypes.c_int64(16384), ctypes.c_int64(64), out, 8)
    Ps = list(out[:k])
    assert Ps[0] >= 64 and all(p >= 2 for p in Ps)
    m = 16384
    for P in Ps:  # every level feasible, last reduced system short
        assert m >= 2 * P - 1
        m = 2 * P - 1
    assert m <= 48
    k = lib().dag_auto_partitions(ctypes.c_int64(365), ctypes.c_int64(2048), out, 8)
    assert list(out[:k]) == [1]


@pytest.mark.parametrize("n,b,a", [(4, 70, 5), (9, 64, 3), (12, 33, 0), (7, 130, 70), (3, 5, 2)])
def test_twisted_selinv_graph(n, b, a, monkeypatch):
    # selinv eliminates the two halves of the chain towards the meeting block
    # (reading R13): same X and log det as Alg. 1 + Alg. 2, different task list
    A0 = btagen.g2(6, n, b, a)
    L, X, ld = seq.selinv(A0)
    counts = {}
    for mode in ("twisted", "one-sided"):
        monkeypatch.setenv("SERINV_OPT", "twist_min_n=3" if mode == "twisted" else "twist_min_n=0")
        A, nn, bb, aa = prep(A0)
        ldv, info, nt = ctypes.c_double(0), ctypes.c_int(0), ctypes.c_int64(0)
        rc = lib().dag_run_sequential(2, ctypes.c_int64(nn), ctypes.c_int64(bb), ctypes.c_int64(aa), *ptrs(A),
                                      ctypes.byref(ldv), ctypes.byref(info), 16, 4, ctypes.byref(nt), -1)
        assert rc == 0 and info.value == 0
        assert inv.max_block_err(cut(A, X), X)[0] < 1e-12, mode
        assert abs(ldv.value - ld) <= 1e-12 * max(1, abs(ld))
        counts[mode] = nt.value
    assert counts["twisted"] != counts["one-sided"]


@pytest.mark.parametrize("n,b,a", [(4, 200, 5), (5, 130, 70), (3, 256, 0), (6, 192, 3)])
def test_wide_tasks(n, b, a, monkeypatch):
    # 128-row GEMM tasks (paired row tiles) for the inversion waves and the L W
    # precompute: forced on for every wave, same results (sequential, twisted, nested)
    monkeypatch.setenv("SERINV_OPT", "wide_min_wave=1")
    A0 = btagen.g2(7, n, b, a)
    L, X, ld = seq.selinv(A0)
    for kind, src, ref in ((2, A0, X), (1, L, X)):
        R, ldr, info = run_seq(kind, src)
        assert info == 0
        assert inv.max_block_err(cut(R, ref), ref)[0] < 1e-12
    if n >= 3:
        rc, R, ldr, info = run_nested(A0, [2])
        assert rc == 0 and info == 0
        assert inv.max_block_err(cut(R, X), X)[0] < 1e-12


def test_plan_ends_policy():
    # serinv_plan_ends (reading R14): both chain ends take r x a middle's blocks
    from paper_2503_17528_b200 import plan, plan_ends
    for n in range(2, 70):
        for P in range(1, 9):
            for r in (0.5, 1.0, 1.7, 3.0):
                if n < 2 * P - 1:
                    continue
                pe = plan_ends(n, P, r)
                assert pe[0][0] == 0 and pe[-1][1] == n
                assert all(pe[i][1] == pe[i + 1][0] for i in range(P - 1))
                assert all(e - s >= 1 for s, e in pe)
                assert all(e - s >= 2 for s, e in pe[1:-1])
                if r == 1.0 and P != 2:
                    assert pe == plan(n, P, 1.0)
                if P == 2:
                    assert pe == [(0, n // 2), (n // 2, n)]
    pe = plan_ends(1024, 8, 1.7)
    assert pe[0][1] - pe[0][0] == pe[-1][1] - pe[-1][0] > pe[1][1] - pe[1][0]


@pytest.mark.parametrize("r", [0.5, 1.7, 2.5])
@pytest.mark.parametrize("P", [3, 4, 6])
def test_pselinv_graph_ends_plan(P, r):
    A0 = btagen.g2(8, 30, 20, 3)
    L, X, ld = seq.selinv(A0)
    A, n, b, a = prep(A0)
    ldv, info, nt = ctypes.c_double(0), ctypes.c_int(0), ctypes.c_int64(0)
    rc = lib().dag_run_pselinv(ctypes.c_int64(n), ctypes.c_int64(b), ctypes.c_int64(a), P, ctypes.c_double(r),
                               *ptrs(A), ctypes.byref(ldv), ctypes.byref(info), 16, ctypes.byref(nt))
    assert rc == 0 and info.value == 0
    assert inv.max_block_err(cut(A, X), X)[0] < 1e-11
    assert abs(ldv.value - ld) <= 1e-12 * max(1, abs(ld))


@pytest.mark.parametrize("P,Q", [(3, 1), (3, 2), (2, 4)])
@pytest.mark.parametrize("where", ["interior", "boundary", "tip"])
def test_distributed_info_is_global_and_agreed(P, Q, where):
    # every rank reports the SAME status after serinv_ppobtasi (dist_meta.h):
    # a bad pivot inside a partition (met by one rank's PPOBTAF), at a partition
    # boundary (met in the redundant reduced solve, whose row labels for other
    # ranks' partitions are decoded from the exchange records), or in the tip.
    # The reported row is the genuine failure (finite pivot <= 0); the NaN pivots it
    # propagates to other blocks are not reported.  dag_run_distributed_q returns -4
    # if two ranks disagree.
    n, b, a = 36, 5, 2
    A0 = btagen.g1(5, n, b, a)
    s1, e1 = par.plan(n, P, 1.0)[1]
    c1 = (e1 - s1) // Q + ((e1 - s1) % Q > 0)    # rank 1's first sub-partition: [s1, s1 + c1)
    assert c1 >= 3
    if where == "interior":
        blk = s1 + 1 if P > 2 else s1 + c1 - 2   # eliminated inside rank 1's PPOBTAF
        A0["diag"][blk][1, 1] = -1e6
        expect = blk * b + 2
    elif where == "boundary":
        blk = s1                                 # a boundary block: met in the reduced system
        A0["diag"][blk][3, 3] = -1e6
        expect = blk * b + 4
    else:
        A0["tip"][1, 1] = -1e6
        expect = n * b + 2
    A, n_, b_, a_ = prep(A0)
    ldv, info = ctypes.c_double(0), ctypes.c_int(0)
    rc = lib().dag_run_distributed_q(ctypes.c_int64(n), ctypes.c_int64(b), ctypes.c_int64(a), P, Q,
                                     ctypes.c_double(1.0), *ptrs(A), ctypes.byref(ldv), ctypes.byref(info))
    assert rc == 0, rc
    assert info.value == expect, (info.value, expect)
    assert np.isnan(ldv.value)


@pytest.mark.parametrize("opt", ["carry_min_b=64", "carry_min_b=64,split_last=1",
                                 "carry_min_b=64,rts1_chain=1,split_last=2,update_group=3",
                                 "carry_min_b=64,twist_min_n=3,twist_max_b=4096"])
def test_carried_chain_options(opt, monkeypatch):
    # carried chain (C3's b >= 2048 default) at small b, with its scheduling options
    # and in the twisted order: same results, valid emission order
    monkeypatch.setenv("SERINV_OPT", opt if "twist" in opt else opt + ",twist_min_n=0")
    for n, b, a in ((5, 200, 3), (5, 192, 3), (4, 128, 0)):
        A0 = btagen.g1(5, n, b, a)
        L, X, ld = seq.selinv(A0)
        R, ldr, info = run_seq(2, A0)
        assert info == 0
        assert inv.max_block_err(cut(R, X), X)[0] < 1e-12
        assert abs(ldr - ld) <= 1e-12 * max(1, abs(ld))
