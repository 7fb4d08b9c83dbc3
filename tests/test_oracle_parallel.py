"""Pins for oracle/parallel.py (§4, eq. partitionsize, eq. KL, eqs. covpool)."""
import json
import math
import os

import numpy as np
import pytest

from oracle.parallel import (choose_q, entrywise_median, feistel_perm, feistel_perm_array,
                             kl_deviation, kl_rank_key, partition, select_and_pool)

G = os.path.join(os.path.dirname(__file__), "golden")


def test_choose_q_table4_panel_c():
    t = json.load(open(os.path.join(G, "table4_panel_c.json")))
    cells = 0
    for n, row in t["rows"].items():
        for (omega, p), q in zip(t["columns"], row):
            assert choose_q(int(n), p, omega) == q, (n, omega, p)
            cells += 1
    assert cells == 90


def test_choose_q_spec_examples_and_cap():
    assert choose_q(2 ** 16, 4, 2 ** 12) == 4
    assert choose_q(2 ** 10, 16, 2 ** 12) == 1
    assert choose_q(2 ** 19, 8, 2 ** 13) == 8
    assert choose_q(8_000_000, 40, 4096) == 48
    assert choose_q(8_000_000, 40, 4096, cap=8) == 8


@pytest.mark.parametrize("n", [2, 3, 5, 10, 17, 1000, 4099, 65536, 100_003])
def test_feistel_is_permutation(n):
    pi = feistel_perm_array(n, seed=12345)
    assert np.array_equal(np.sort(pi), np.arange(n))


def test_feistel_scalar_equals_vector_and_seeded():
    n = 5000
    v = feistel_perm_array(n, seed=77)
    assert all(feistel_perm(i, n, 77) == v[i] for i in range(0, n, 37))
    assert not np.array_equal(v, feistel_perm_array(n, seed=78))
    assert np.array_equal(v, feistel_perm_array(n, seed=77))


def test_partition_sizes():
    block, pos, m = partition(10, 3, seed=1)
    assert m == 3 and np.sum(block == -1) == 1
    for l in range(3):
        assert sorted(pos[block == l]) == [0, 1, 2]
    b1, p1, m1 = partition(10, 1, seed=1)
    assert m1 == 10 and np.array_equal(p1, np.arange(10))


def test_median_examples():
    D = [np.diag([1.0, 1.0]), np.diag([2.0, 2.0]), np.diag([9.0, 9.0])]
    assert np.array_equal(entrywise_median(D), np.diag([2.0, 2.0]))
    assert np.array_equal(entrywise_median([np.ones(2), 3 * np.ones(2)]), 2 * np.ones(2))


def test_kl_examples():
    I2 = np.eye(2)
    assert kl_deviation(np.zeros(2), I2, np.zeros(2), I2) == pytest.approx(0.0, abs=1e-15)
    assert kl_deviation(np.zeros(1), np.array([[2.0]]), np.zeros(1), np.array([[1.0]])) == \
        pytest.approx(1 - math.log(2), rel=1e-14)
    assert kl_deviation(np.array([1.0, 0]), I2, np.zeros(2), I2) == pytest.approx(1.0, rel=1e-14)
    rng = np.random.default_rng(0)
    A = rng.standard_normal((4, 4))
    S = A @ A.T + np.eye(4)
    assert kl_deviation(np.zeros(4), 2 * S, np.zeros(4), S) == pytest.approx(4 * (1 - math.log(2)), rel=1e-12)


def test_kl_rank_key_orders_like_kl():
    rng = np.random.default_rng(1)
    mus, Ss = [], []
    for _ in range(7):
        A = rng.standard_normal((3, 3))
        Ss.append(A @ A.T + np.eye(3))
        mus.append(rng.standard_normal(3))
    mm, Sm = entrywise_median(mus), entrywise_median(Ss)
    kl = [kl_deviation(mm, Sm, mus[l], Ss[l]) for l in range(7)]
    key = [kl_rank_key(mm, Sm, mus[l], Ss[l]) for l in range(7)]
    assert np.argsort(kl).tolist() == np.argsort(key).tolist()


def test_pooling_equals_concatenation():
    # pooled moments = classical moments of the concatenated sets
    rng = np.random.default_rng(2)
    m = 400
    sets = [rng.standard_normal((m, 3)) * (l + 1) + l for l in range(3)]
    mus = [s.mean(0) for s in sets]
    Ss = [np.cov(s, rowvar=False) for s in sets]
    # make all three kept: q = 3 keeps ceil(3/2) = 2, so use q = 1.. pool all by duplicating ranks
    mu_p, S_p, kept, _ = select_and_pool(mus + mus[:0], Ss, [m] * 3)
    allrows = np.concatenate([sets[k] for k in kept])
    assert np.allclose(mu_p, allrows.mean(0), rtol=1e-12)
    assert np.allclose(S_p, np.cov(allrows, rowvar=False), rtol=1e-10)


def test_majority_identical_recovers_exactly():
    # a strict majority of identical fits -> pooled = that fit
    rng = np.random.default_rng(3)
    mu = rng.standard_normal(3)
    A = rng.standard_normal((3, 3))
    S = A @ A.T + np.eye(3)
    mus = [mu] * 5 + [mu + 10, mu - 7]
    Ss = [S] * 5 + [S * 9, S + 4 * np.eye(3)]
    mu_p, S_p, kept, _ = select_and_pool(mus, Ss, [1000] * 7)
    assert set(kept) <= {0, 1, 2, 3, 4} and len(kept) == 4
    # eqs. covpool with weights m and denominator n_pooled - 1 (verbatim, R15):
    # four identical fits give Lambda = 4 (m-1) S over n_pooled = 4 m
    assert np.allclose(mu_p, mu, rtol=1e-14)
    assert np.allclose(S_p, S * (4 * 999) / (4 * 1000 - 1), rtol=1e-13)


def test_single_block_is_identity():
    rng = np.random.default_rng(4)
    A = rng.standard_normal((3, 3))
    S = A @ A.T
    mu = rng.standard_normal(3)
    mu_p, S_p, kept, _ = select_and_pool([mu], [S], [77])
    assert np.array_equal(mu_p, mu) and np.allclose(S_p, S, rtol=1e-15)


def test_contiguous_partition():
    block, pos, m = partition(10, 3, seed=1, mode="contiguous")
    assert m == 3 and list(block) == [0, 0, 0, 1, 1, 1, 2, 2, 2, -1] and list(pos[:9]) == [0, 1, 2] * 3
