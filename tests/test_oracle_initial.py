"""Pins for oracle/initial.py (eq. wrapping, eq. LR; SPEC.md:218-254 examples)."""
import json
import math
import os

import numpy as np
import pytest

from oracle.initial import (DegenerateNorms, gsscm_lr, lr_cutoffs, row_norms, wrap,
                            wrapped_covariance, xi)

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))
W = GOLD["wrapping"]


def test_wrap_values():
    assert wrap(np.array([0.0]))[0] == 0.0
    assert wrap(np.array([1.0]))[0] == 1.0
    assert wrap(np.array([1.5]))[0] == 1.5                    # identity branch includes b
    z = 1.5 + 1e-12
    assert wrap(np.array([z]))[0] == pytest.approx(W["q1"] * math.tanh(W["q2"] * (W["c"] - z)), rel=1e-15)
    assert wrap(np.array([4.0]))[0] == 0.0                    # q1 tanh(0) = 0 at |z| = c
    assert wrap(np.array([5.0]))[0] == 0.0
    assert wrap(np.array([-2.5]))[0] == pytest.approx(-W["q1"] * math.tanh(W["q2"] * 1.5), rel=1e-15)


def test_wrap_odd_bounded():
    z = np.linspace(-10, 10, 20001)
    g = wrap(z)
    assert np.array_equal(wrap(-z), -g)
    assert np.max(np.abs(g)) <= W["q1"]


def test_wrapped_cov_identity_branch_is_classical():
    rng = np.random.default_rng(0)
    Z = np.clip(rng.standard_normal((500, 4)), -1.5, 1.5)
    assert np.allclose(wrapped_covariance(Z), np.cov(Z, rowvar=False), rtol=1e-13, atol=1e-15)


def test_wrapped_cov_far_row_equals_zero_row():
    rng = np.random.default_rng(1)
    Z = rng.standard_normal((300, 3))
    A = Z.copy(); A[7] = 1e6
    B = Z.copy(); B[7] = 0.0
    assert np.array_equal(wrapped_covariance(A), wrapped_covariance(B))


def test_lr_cutoffs_example():
    g = GOLD["spec_examples"]["lr_cutoffs"]
    A, B = lr_cutoffs(np.array(g["norms"], float))
    assert (A, B) == (g["A"], g["B"])
    with pytest.raises(DegenerateNorms):
        lr_cutoffs(np.ones(10))
    A2, B2 = lr_cutoffs(3.0 * np.array(g["norms"], float))
    assert (A2, B2) == (3 * A, 3 * B)


def test_xi_branches():
    r = np.array([0.0, 3.0, 4.5, 6.0, 7.0])
    assert np.allclose(xi(r, 3.0, 6.0), [1, 1, 0.5, 0, 0])


def test_gsscm_all_inside_is_second_moment():
    # all rows with ||z|| <= A -> xi = 1; construct norms so that every norm equals A
    rng = np.random.default_rng(2)
    U = rng.standard_normal((101, 3))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    r = np.linspace(1.0, 2.0, 101)
    Z = U * r[:, None]
    S = gsscm_lr(Z)
    A, B = lr_cutoffs(row_norms(Z))
    w = np.where(row_norms(Z) <= A, 1.0, np.where(row_norms(Z) <= B, (B - row_norms(Z)) / (B - A), 0.0))
    expect = sum(w[i] ** 2 * np.outer(Z[i], Z[i]) for i in range(101)) / 101
    assert np.allclose(S, expect, rtol=1e-13)


def test_gsscm_hand_example():
    # n = 5, p = 2; norms 1..5 on the axes -> A = 3, B = 6; xi = 1,1,1,2/3,1/3
    Z = np.array([[1.0, 0], [0, 2.0], [3.0, 0], [0, 4.0], [5.0, 0]])
    S = gsscm_lr(Z)
    e00 = (1 + 9 + (1 / 3) ** 2 * 25) / 5
    e11 = (4 + (2 / 3) ** 2 * 16) / 5
    assert np.allclose(S, [[e00, 0], [0, e11]], rtol=1e-15)


def test_gsscm_far_row_contributes_zero():
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((400, 3))
    A = Z.copy(); A[5] = 1e3   # norm far beyond B, and B is unchanged (its rank position is the same)
    B = Z.copy(); B[5] = 1e4
    assert np.allclose(gsscm_lr(A), gsscm_lr(B), rtol=0, atol=0)


def test_row_permutation_invariance():
    rng = np.random.default_rng(4)
    Z = rng.standard_normal((1000, 5))
    P = rng.permutation(1000)
    assert np.allclose(wrapped_covariance(Z[P]), wrapped_covariance(Z), rtol=1e-13)
    assert np.allclose(gsscm_lr(Z[P]), gsscm_lr(Z), rtol=1e-13)
