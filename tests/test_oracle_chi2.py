"""Pins for oracle/chi2.py against closed forms (not the library routine it calls)."""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import ndtri

from oracle.chi2 import chi2_cdf, chi2_quantile, consistency_factor

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))
PROBS = [0.01, 0.25, 0.5, 0.75, 0.9, 0.975, 0.999]


@pytest.mark.parametrize("u", PROBS)
def test_quantile_p2_closed_form(u):
    # F_2(x) = 1 - exp(-x/2)  =>  chi2_{2,u} = -2 ln(1-u)
    assert chi2_quantile(u, 2) == pytest.approx(-2.0 * math.log1p(-u), rel=1e-13)


@pytest.mark.parametrize("u", PROBS)
def test_quantile_p1_normal(u):
    # chi2_1 = Z^2  =>  chi2_{1,u} = (Phi^-1((1+u)/2))^2
    assert chi2_quantile(u, 1) == pytest.approx(ndtri(0.5 * (1.0 + u)) ** 2, rel=1e-12)


def _poisson_cdf_even(x, p):
    # even p = 2k: F(x) = 1 - exp(-x/2) sum_{j<k} (x/2)^j / j!
    k = p // 2
    t = x / 2.0
    return 1.0 - math.exp(-t) * sum(t ** j / math.factorial(j) for j in range(k))


@pytest.mark.parametrize("p", [2, 4, 8, 10, 16, 20, 40])
@pytest.mark.parametrize("u", [0.5, 0.75, 0.975])
def test_even_dof_poisson_sum(p, u):
    x = chi2_quantile(u, p)
    assert _poisson_cdf_even(x, p) == pytest.approx(u, abs=1e-13)
    assert chi2_cdf(x, p) == pytest.approx(u, abs=1e-13)


@pytest.mark.parametrize("p", [1, 3, 5, 7])
def test_odd_dof_recurrence(p):
    # F_{p+2}(x) = F_p(x) - (x/2)^{p/2} e^{-x/2} / Gamma(p/2 + 1); F_1(x) = erf(sqrt(x/2))
    x = 7.3
    F = math.erf(math.sqrt(x / 2))
    for d in range(1, p, 2):
        F -= (x / 2) ** (d / 2) * math.exp(-x / 2) / math.gamma(d / 2 + 1)
    assert chi2_cdf(x, p) == pytest.approx(F, abs=1e-14)


def test_spec_examples():
    for dof, prob, val in GOLD["spec_examples"]["chi2_quantile"]:
        assert chi2_quantile(prob, dof) == pytest.approx(val, abs=5e-6 * max(1, val))
    assert chi2_quantile(1 - math.exp(-1), 2) == pytest.approx(2.0, rel=1e-14)


def test_quantile_monotone():
    for p in (1, 5, 40):
        xs = [chi2_quantile(u, p) for u in np.linspace(0.01, 0.99, 50)]
        assert all(b > a for a, b in zip(xs, xs[1:]))


@pytest.mark.parametrize("alpha", [0.5, 0.5000010, 0.6, 0.75, 0.9, 0.975])
def test_consistency_p2_closed_form(alpha):
    # F_4(chi2_{2,a}) = 1 - (1-a)(1 - ln(1-a))
    expect = alpha / (1.0 - (1.0 - alpha) * (1.0 - math.log1p(-alpha)))
    assert consistency_factor(alpha, 2) == pytest.approx(expect, rel=1e-13)


@pytest.mark.parametrize("alpha", [0.5, 0.6, 0.75, 0.975])
def test_consistency_p1_truncated_normal(alpha):
    # variance of N(0,1) truncated to |z| <= q, q = Phi^-1((1+a)/2): (a - 2 q phi(q)) / a
    q = ndtri(0.5 * (1 + alpha))
    phi = math.exp(-0.5 * q * q) / math.sqrt(2 * math.pi)
    assert consistency_factor(alpha, 1) == pytest.approx(alpha / (alpha - 2 * q * phi), rel=1e-12)


@pytest.mark.parametrize("p", [4, 5, 8, 10, 20, 40])
@pytest.mark.parametrize("alpha", [0.5, 0.75, 0.975])
def test_consistency_general_recurrence(p, alpha):
    # F_{p+2}(q) = F_p(q) - (q/2)^{p/2} e^{-q/2} / Gamma(p/2+1) with F_p(q) = alpha
    q = chi2_quantile(alpha, p)
    Fp2 = alpha - math.exp((p / 2) * math.log(q / 2) - q / 2 - math.lgamma(p / 2 + 1))
    assert consistency_factor(alpha, p) == pytest.approx(alpha / Fp2, rel=1e-12)


def test_consistency_full_sample():
    for p in (1, 7, 40):
        assert consistency_factor(1.0, p) == 1.0


def test_consistency_monte_carlo_p3():
    # c(a,p) * E[x x^T | x^T x <= chi2_{p,a}] = I for x ~ N(0, I_p)
    rng = np.random.default_rng(5)
    G = rng.standard_normal((400_000, 3))
    a = 0.75
    keep = np.einsum("ij,ij->i", G, G) <= chi2_quantile(a, 3)
    v = np.mean(G[keep] ** 2)
    assert consistency_factor(a, 3) * v == pytest.approx(1.0, abs=0.01)
