"""Pins for oracle/parallel.py (PPOBTAF / POBTARSSI / PPOBTASI, Sec. 3) -- CPU only.

The partitioned pipeline must return the dense inverse on the pattern for any
P and r ("true inverse boundary blocks"), with n_r = 2P-1
(P:513), and reproduce Fig. 2's partition of n = 11 into 3.
Mutation tests show the G2 generator makes a dropped fill-in term visible.
"""
import inspect
import os
import textwrap

import numpy as np
import pytest

import btagen
from oracle import dense, invariants as inv, parallel as par, sequential as seq

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    with open(os.path.join(GOLD, name)) as f:
        return [l.split() for l in f if l.strip() and not l.startswith("#")]


def test_fig2_partition_golden():
    for n, P, r, first1, first1_perm in _rows("fig2_partition.txt"):
        parts = par.plan(int(n), int(P), float(r))
        assert parts[1][0] == int(first1)
        # after the implicit shifting permutation the first eliminated block is s+1
        assert parts[1][0] + 1 == int(first1_perm)


def test_reduced_size_golden():
    for P, nr in _rows("reduced_size.txt"):
        P, nr = int(P), int(nr)
        n = max(2 * P - 1, 3 * P)
        A = btagen.g1(1, n, 2, 1)
        R = par.pselinv(A, P)
        assert R["Ar"]["diag"].shape[0] == nr == 2 * P - 1


def test_plan_properties():
    for n in range(1, 60):
        for P in range(1, 9):
            for r in (0.5, 1.0, 1.8, 2.25, 4.0):
                if n < 2 * P - 1:
                    with pytest.raises(par.TooFewBlocks):
                        par.plan(n, P, r)
                    continue
                parts = par.plan(n, P, r)
                assert parts[0][0] == 0 and parts[-1][1] == n
                for p in range(P - 1):
                    assert parts[p][1] == parts[p + 1][0]
                assert parts[0][1] - parts[0][0] >= 1
                sizes = [e - s for s, e in parts[1:]]
                assert all(s >= 2 for s in sizes)
                if sizes:
                    assert max(sizes) - min(sizes) <= 1
                    assert sizes == sorted(sizes, reverse=True)   # remainder to earlier middles


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("gen", ["g1", "g2"])
def test_pselinv_matches_dense_and_sequential(P, gen):
    for (n, b, a) in [(2 * P - 1, 3, 2), (3 * P + 1, 4, 2), (5 * P, 3, 0), (4 * P + 3, 2, 3)]:
        A = btagen.generate(gen, 7 + P, n, b, a)
        R = par.pselinv(A, P)
        Xd = dense.dense_inverse_pattern(A)
        e, where = inv.max_block_err(R["X"], Xd)
        assert e < 1e-11, (n, b, a, e, where)
        ldd = dense.dense_logdet(A)
        assert abs(R["logdet"] - ldd) <= 1e-12 * max(1.0, abs(ldd))
        # eliminated blocks of the top partition equal the sequential factor (prefix property)
        Ls = seq.pobtaf(A)
        for i in range(R["parts"][0][1] - 1):
            assert inv.rel_err(R["L"]["diag"][i], Ls["diag"][i]) < 1e-14
            assert inv.rel_err(R["L"]["lower"][i], Ls["lower"][i]) < 1e-14


def test_p1_is_sequential():
    A = btagen.g2(4, 9, 4, 2)
    R = par.pselinv(A, 1)
    L, X, ld = seq.selinv(A)
    assert inv.max_block_err(R["X"], X)[0] < 1e-14
    assert abs(R["logdet"] - ld) < 1e-12 * abs(ld)


def test_values_independent_of_ratio():
    A = btagen.g2(5, 30, 3, 2)
    ref = par.pselinv(A, 4, 1.0)["X"]
    for r in (0.5, 1.8, 2.25, 3.0):
        X = par.pselinv(A, 4, r)["X"]
        assert inv.max_block_err(X, ref)[0] < 1e-12


def test_middle_partition_of_two_blocks():
    # smallest middles (loop bodies of Alg. 4/6 empty): everything lands in A_r
    A = btagen.g2(6, 7, 3, 2)
    R = par.pselinv(A, 4, 0.1)
    assert [e - s for s, e in R["parts"]] == [1, 2, 2, 2]
    assert inv.max_block_err(R["X"], dense.dense_inverse_pattern(A))[0] < 1e-12


def _mutant(func, tag):
    """Copy of `func` with the source line carrying comment `# <tag>` removed."""
    src = textwrap.dedent(inspect.getsource(func))
    lines = src.splitlines()
    hit = [i for i, l in enumerate(lines) if l.rstrip().endswith("# " + tag)]
    assert len(hit) == 1, tag
    indent = lines[hit[0]][: len(lines[hit[0]]) - len(lines[hit[0]].lstrip())]
    lines[hit[0]] = indent + "pass"
    ns = dict(par.__dict__)
    exec("\n".join(lines), ns)
    return ns[func.__name__]


@pytest.mark.parametrize("func,tag", [
    ("permuted_pobtaf", "l.10"), ("permuted_pobtaf", "l.11"), ("permuted_pobtaf", "l.12"),
    ("permuted_pobtaf", "l.9"),
    ("permuted_pobtasi", "l.3"), ("permuted_pobtasi", "l.8"), ("permuted_pobtasi", "l.11"),
])
def test_mutations_of_fill_in_terms_are_detected(func, tag):
    # Dropping any fill-in term of Alg. 4 / Alg. 6 must fail the dense pin on G2 data
    # (G1's fast fill-in decay hides them; G2 decays ~0.73 per block).
    A = btagen.g2(11, 26, 6, 2)
    Xd = dense.dense_inverse_pattern(A)
    orig = getattr(par, func)
    try:
        setattr(par, func, _mutant(orig, tag))
        R = par.pselinv(A, 3)
    except seq.NotPositiveDefinite:
        return                      # detected: the mutated reduced system is not SPD
    finally:
        setattr(par, func, orig)
    e, where = inv.max_block_err(R["X"], Xd)
    assert e > 1e-6, (func, tag, e)
    # and a majority of the middle partitions' blocks are flagged
    bad = 0
    tot = 0
    for p in range(1, 3):
        s, e_ = R["parts"][p]
        for i in range(s, e_):
            tot += 1
            bad += inv.rel_err(R["X"]["diag"][i], Xd["diag"][i]) > 1e-10
    assert bad >= 1


def test_tip_accumulators_sum_to_sequential_downdate():
    # Alg. 3 l.8: A_nn + sum U_p is the tip after all arrow eliminations of the partitions
    A = btagen.g1(3, 12, 2, 1)
    R = par.pselinv(A, 2)
    U = R["U"][0] + R["U"][1]
    assert U.shape == (1, 1) and U[0, 0] < 0
