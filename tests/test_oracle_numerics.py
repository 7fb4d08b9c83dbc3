"""Pins for oracle/numerics.py (SPEC.md:43-99 examples, hand formulas)."""
import math

import numpy as np
import pytest
from scipy.linalg import solve_triangular

from oracle.numerics import (NotPositiveDefinite, cholesky, cond1, eigh_desc, logdet_from_chol,
                             mahalanobis_sq)


def test_cholesky_examples():
    assert np.allclose(cholesky(np.eye(3)), np.eye(3))
    assert np.allclose(cholesky(np.diag([4.0, 9.0])), np.diag([2.0, 3.0]))
    with pytest.raises(NotPositiveDefinite):
        cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_logdet_examples():
    assert logdet_from_chol(np.eye(4)) == 0.0
    assert logdet_from_chol(np.diag([2.0, 3.0])) == pytest.approx(math.log(36.0), rel=1e-15)
    assert logdet_from_chol(np.diag([1e-6, 1e-6])) == pytest.approx(4 * math.log(1e-6), rel=1e-14)


def test_logdet_vs_cofactor():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((3, 3))
    S = A @ A.T + np.eye(3)
    det = (S[0, 0] * (S[1, 1] * S[2, 2] - S[1, 2] * S[2, 1])
           - S[0, 1] * (S[1, 0] * S[2, 2] - S[1, 2] * S[2, 0])
           + S[0, 2] * (S[1, 0] * S[2, 1] - S[1, 1] * S[2, 0]))
    assert math.exp(logdet_from_chol(cholesky(S))) == pytest.approx(det, rel=1e-12)


def test_cond1_examples():
    assert cond1(np.eye(3)) == 1.0
    assert cond1(np.diag([1000.0, 1.0])) == pytest.approx(1000.0, rel=1e-15)
    assert cond1(np.diag([1.0, 1e-4])) == pytest.approx(1e4, rel=1e-12)
    rng = np.random.default_rng(1)
    A = rng.standard_normal((5, 5))
    S = A @ A.T + np.eye(5)
    assert cond1(7.5 * S) == pytest.approx(cond1(S), rel=1e-12)
    # 2x2 by hand: inverse of [[a,b],[b,d]] = [[d,-b],[-b,a]]/(ad-b^2)
    a, b, d = 3.0, 1.0, 2.0
    S2 = np.array([[a, b], [b, d]])
    inv1 = max(abs(d) + abs(b), abs(b) + abs(a)) / (a * d - b * b)
    assert cond1(S2) == pytest.approx(max(a + b, b + d) * inv1, rel=1e-14)


def test_eigen_examples():
    w, V = eigh_desc(np.diag([1.0, 3.0]))
    assert np.allclose(w, [3.0, 1.0])
    assert np.allclose(np.abs(V), [[0, 1], [1, 0]])
    w, V = eigh_desc(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(w, [3.0, 1.0])
    assert np.allclose(np.abs(V[:, 0]), [1 / math.sqrt(2)] * 2)
    assert np.allclose(np.abs(V[:, 1]), [1 / math.sqrt(2)] * 2)
    rng = np.random.default_rng(2)
    A = rng.standard_normal((6, 6))
    S = A @ A.T
    w, V = eigh_desc(S)
    assert np.all(np.diff(w) <= 0)
    assert np.allclose(V @ np.diag(w) @ V.T, S, atol=1e-12)
    assert np.allclose(V.T @ V, np.eye(6), atol=1e-13)


def test_mahalanobis_examples():
    Z = np.array([[3.0, 4.0], [1.0, 0.0]])
    assert np.allclose(mahalanobis_sq(Z, np.zeros(2), np.eye(2)), [25.0, 1.0])
    assert mahalanobis_sq(np.array([[2.0]]), np.zeros(1), np.array([[4.0]]))[0] == pytest.approx(1.0)


def test_mahalanobis_equals_cholesky_solve():
    # d = ||L^-1 (z - mu)|| (eq. cholesky), computed independently
    rng = np.random.default_rng(3)
    A = rng.standard_normal((3, 3))
    S = A @ A.T + 0.5 * np.eye(3)
    mu = rng.standard_normal(3)
    Z = rng.standard_normal((50, 3))
    L = np.linalg.cholesky(S)
    Y = solve_triangular(L, (Z - mu).T, lower=True)
    assert np.allclose(mahalanobis_sq(Z, mu, S), np.sum(Y * Y, axis=0), rtol=1e-12)
