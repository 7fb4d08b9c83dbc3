"""Pins for oracle/refine.py and oracle/cstep.py (§3.3, §2.1, §3.5)."""
import numpy as np
import pytest

from oracle.cstep import SingularCandidate, concentrate, delta_update, h_subset, mean_cov
from oracle.numerics import mahalanobis_sq
from oracle.refine import IllConditioned, refine
from paper_1910_05615_b200 import datagen


def test_refine_identity_start_on_gaussian():
    # S_init = I, standard Gaussian -> Sigma ~ I, mu ~ 0
    Z = datagen.gaussian(100_000, 4, seed=1)
    r = refine(np.eye(4), Z)
    assert np.allclose(r.Sigma, np.eye(4), atol=0.05)
    assert np.allclose(r.mu, 0, atol=0.02)


def test_refine_ill_conditioned():
    Z = datagen.gaussian(2000, 2, seed=2)
    with pytest.raises(IllConditioned):
        refine(np.diag([1.0, 1e-6]), Z)
    Zd = datagen.gaussian(2000, 3, seed=3)
    Zd[:, 2] = Zd[:, 1]
    with pytest.raises(IllConditioned):
        refine(np.cov(Zd, rowvar=False), Zd)


def test_refine_keeps_eigenvectors():
    # only the eigenvalues change
    rng = np.random.default_rng(4)
    Q, _ = np.linalg.qr(rng.standard_normal((5, 5)))
    S = (Q * np.array([5.0, 3.0, 2.0, 1.0, 0.5])) @ Q.T
    Z = datagen.gaussian(20_000, 5, seed=5, sigma=S)
    r = refine(S, Z)
    M = r.V.T @ np.linalg.eigh(r.Sigma)[1]
    assert np.allclose(np.sort(np.abs(M).max(axis=0)), 1.0, atol=1e-8)


def test_refine_sphering_roundtrip():
    Z = datagen.gaussian(5000, 3, seed=6)
    r = refine(np.cov(Z, rowvar=False), Z)
    w, V = np.linalg.eigh(r.Sigma)
    Smh = (V / np.sqrt(w)) @ V.T
    assert np.allclose(Smh @ r.Sigma @ Smh, np.eye(3), atol=1e-10)
    assert np.allclose(r.Sigma, (r.V * r.dtilde) @ r.V.T, rtol=1e-13)


def _start(Z):
    return Z.mean(0) + 0.3, np.cov(Z, rowvar=False) * 2.0


@pytest.mark.parametrize("seed", range(4))
def test_cstep_determinant_monotone(seed):
    # det(Sigma_new) <= det(Sigma_old)
    d = datagen.make_config(1 + (seed % 2), n=3000)
    Z = d.X
    mu0, S0 = _start(Z)
    r = concentrate(Z, mu0, S0, d.h)
    ld = [np.linalg.slogdet(S0)[1]] + r.logdets
    assert all(b <= a + 1e-12 for a, b in zip(ld, ld[1:]))
    assert r.converged


def test_cstep_fixed_point_stable():
    d = datagen.make_config(1)
    r = concentrate(d.X, *_start(d.X), d.h)
    r2 = concentrate(d.X, r.mu, r.Sigma, d.h)
    # one C-step reproduces H, the second confirms convergence
    assert np.array_equal(r2.H, r.H) and r2.steps == 2 and r2.logdets == [r.logdet]


def test_cstep_h_equals_n_is_classical():
    Z = datagen.gaussian(500, 3, seed=7)
    r = concentrate(Z, np.ones(3), 4 * np.eye(3), 500)
    assert np.allclose(r.mu, Z.mean(0), rtol=1e-14)
    assert np.allclose(r.Sigma, np.cov(Z, rowvar=False), rtol=1e-13)
    assert r.steps == 2


def test_cstep_condition_monitor():
    Z = datagen.gaussian(200, 2, seed=8)
    with pytest.raises(SingularCandidate):
        concentrate(Z, np.zeros(2), np.diag([1.0, 1e-4]), 150)


def test_h_subset_tie_rule():
    d2 = np.array([3.0, 1.0, 2.0, 2.0, 2.0, 5.0])
    assert list(h_subset(d2, 3)) == [1, 2, 3]


@pytest.mark.parametrize("seed", range(3))
def test_delta_update_equals_recompute(seed):
    # the one-pass update loop gives the new mean and sscp exactly
    rng = np.random.default_rng(seed)
    Z = rng.standard_normal((300, 4)) * [1, 2, 3, 4] + 1.5
    H_old = np.sort(rng.choice(300, 200, replace=False))
    H_new = np.sort(rng.choice(300, 200, replace=False))
    mu_o, S_o = mean_cov(Z, H_old)
    mu_n, S_n = mean_cov(Z, H_new)
    mu_u, Lam_u = delta_update(Z, H_old, H_new, mu_o, (200 - 1) * S_o)
    assert np.allclose(mu_u, mu_n, rtol=1e-11, atol=1e-12)
    assert np.allclose(Lam_u / 199, S_n, rtol=1e-10, atol=1e-12)


def test_mahalanobis_invariant_under_affine():
    # RD invariant under x -> A x + b with (mu, Sigma) transformed along
    rng = np.random.default_rng(9)
    Z = rng.standard_normal((50, 3))
    A = rng.standard_normal((3, 3)) + 3 * np.eye(3)
    b = rng.standard_normal(3)
    mu, S = Z.mean(0), np.cov(Z, rowvar=False)
    d1 = mahalanobis_sq(Z, mu, S)
    d2 = mahalanobis_sq(Z @ A.T + b, A @ mu + b, A @ S @ A.T)
    assert np.allclose(d1, d2, rtol=1e-10)


def test_refine_translation_equivariance_nonidentity():
    # PAPER.md:594-605 (§3.3 step 4): Z~ = Z Sigma_k^{-1/2} and mu_k = Sigma_k^{1/2} mu~.  The univariate
    # MCD is translation equivariant and the scores' scales are not, so refine(S, Z + a) = (mu + a, Sigma).
    # With a non-identity Sigma_k, the wrong back-transform (Sigma^{-1/2} instead of Sigma^{1/2}) gives
    # mu + Sigma^{-1} a instead.
    rng = np.random.default_rng(31)
    Q, _ = np.linalg.qr(rng.standard_normal((4, 4)))
    S = (Q * np.array([9.0, 4.0, 1.0, 0.25])) @ Q.T
    Z = datagen.gaussian(20_000, 4, seed=32, sigma=S)
    a = np.array([3.0, -2.0, 0.5, 7.0])
    r0 = refine(S, Z)
    r1 = refine(S, Z + a)
    assert np.abs(np.diag(r0.Sigma) - 1.0).max() > 0.5          # far from the identity
    assert np.allclose(r1.mu, r0.mu + a, rtol=0, atol=1e-9)
    assert np.allclose(r1.Sigma, r0.Sigma, rtol=1e-9)
    # scale equivariance: refine(S, c Z) = (c mu, c^2 Sigma) for c a power of two (exact)
    r2 = refine(S, 4.0 * Z)
    assert np.allclose(r2.mu, 4.0 * r0.mu, rtol=1e-12, atol=1e-13)
    assert np.allclose(r2.Sigma, 16.0 * r0.Sigma, rtol=1e-12)


def test_refine_p1_is_the_reweighted_univariate_mcd():
    # p = 1: V = [1], T = Z, Sigma = sigma_uni^2(Z), mu = sigma * mu_uni(Z / sigma) = mu_uni(Z).  Reading R8
    # ("univariate MCD" = the reweighted estimator of §3.1).  SPEC.md:164's worked
    # example x = (0,1,2,3,4,1000): the reweighted MCD keeps {0..4}, so mu = 2 and
    # Sigma = c(0.975,1) * 2.5 with c(0.975,1) = 1.174778641565 (pinned in
    # tests/test_oracle_chi2.py).  The raw estimator would give mu = 1.5 (window {0,1,2,3}, lowest start).
    Z = np.array([0.0, 1.0, 2.0, 3.0, 4.0, 1000.0])[:, None]
    r = refine(np.eye(1), Z)
    assert r.mu[0] == pytest.approx(2.0, rel=1e-14)
    assert r.Sigma[0, 0] == pytest.approx(1.174778641565 * 2.5, rel=1e-11)
