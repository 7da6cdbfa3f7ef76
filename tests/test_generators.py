"""Input generators (btagen): symmetry, SPD, determinism, exact diagonal sums."""
import numpy as np
import pytest

import btagen
from oracle import dense


@pytest.mark.parametrize("gen", ["g1", "g2", "g2k"])
def test_spd_and_symmetric(gen):
    for (n, b, a) in [(8, 4, 2), (5, 7, 0), (3, 5, 6), (1, 1, 1)]:
        A = btagen.generate(gen, 3, n, b, a)
        D = dense.to_dense(A)
        for i in range(n):
            np.testing.assert_array_equal(A["diag"][i], A["diag"][i].T)
        np.testing.assert_array_equal(A["tip"], A["tip"].T)
        assert np.linalg.eigvalsh(D).min() > 0


@pytest.mark.parametrize("gen", ["g1", "g2", "g2k"])
def test_deterministic_and_seed_dependent(gen):
    A = btagen.generate(gen, 4, 6, 5, 2)
    B = btagen.generate(gen, 4, 6, 5, 2)
    C = btagen.generate(gen, 5, 6, 5, 2)
    for k in ("diag", "lower", "arrow", "tip"):
        np.testing.assert_array_equal(A[k], B[k])
    assert not np.array_equal(A["diag"], C["diag"])


def test_g1_diagonal_is_exact_row_sum_in_any_order():
    A = btagen.g1(2, 6, 9, 3)
    D = dense.to_dense(A)
    N = D.shape[0]
    rng = np.random.default_rng(0)
    for r in range(N):
        off = np.abs(np.delete(D[r], r))
        s1 = 0.0
        for v in off:
            s1 += v
        s2 = 0.0
        for v in off[rng.permutation(off.size)]:
            s2 += v
        assert s1 == s2 == D[r, r] - 1.0
    # entries are multiples of 2^-23 in [-1, 1)
    off = D[~np.eye(N, dtype=bool)]
    assert np.all(off * 2 ** 23 == np.round(off * 2 ** 23))
    assert off.min() >= -1.0 and off.max() < 1.0


def test_g2_fill_in_decay_is_slow():
    # fill-in decay ~ root of x^2 - (2+tau) x + 1 ~ 0.73 per block
    tau = 0.1
    x = ((2 + tau) - np.sqrt((2 + tau) ** 2 - 4)) / 2
    assert 0.70 < x < 0.76


def test_bytes():
    assert btagen.bta_bytes(8, 4, 2) == 8 * (8 * 16 + 7 * 16 + 8 * 8 + 4)


def test_torch_twin_of_g1_is_bit_identical():
    import torch
    for (n, b, a, seed) in [(5, 7, 3, 1), (3, 16, 0, 9), (2, 5, 4, 12345)]:
        A = btagen.g1(seed, n, b, a)
        T = btagen.g1_torch(seed, n, b, a, device="cpu")
        for k in ("diag", "lower", "arrow", "tip"):
            assert np.array_equal(A[k], T[k].numpy()), k
        # rank-local slices
        for (s, e) in [(0, 2), (1, n), (1, 3)] if n > 3 else [(0, n)]:
            Tl = btagen.g1_torch(seed, n, b, a, device="cpu", start=s, end=e)
            assert np.array_equal(Tl["diag"].numpy(), A["diag"][s:e])
            nl = e - s - 1 if e == n else e - s
            assert np.array_equal(Tl["lower"].numpy(), A["lower"][s:s + nl])
            assert np.array_equal(Tl["arrow"].numpy(), A["arrow"][s:e])
            assert np.array_equal(Tl["tip"].numpy(), A["tip"])
