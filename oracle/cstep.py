"""Concentration steps (oracle; test infrastructure only).

PAPER.md:255-292 (§2.1, eqs. cstep1-cstep4b): given (mu_old, Sigma_old)
  1. d_old(i) = d(x_i, mu_old, Sigma_old) for all n rows;
  2. sort the distances; 3. H_new = the h smallest;
  4. mu_new = mean of H_new, Sigma_new = covariance of H_new (denominator h-1).
PAPER.md:293-301: det(Sigma_new) <= det(Sigma_old) (pinned as a property).
PAPER.md:643-657 (§3.4): if ||Sigma_old||_1 ||Sigma_old^-1||_1 >= kappa_max the
  C-step is not taken (reading R10: the start is dropped).
PAPER.md:659-713 (§3.5): the update-based loop reaches exactly the same
  (mu_new, Lambda_new) as the recompute — the oracle uses the plain recompute;
  `delta_update` writes the paper's sequential loop out for the pin that the
  two agree.
Readings: R11 ties at the h-th distance broken by row position (the original
  row index when q = 1); R12 stop when H_new == H_old, cap 100 C-steps.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .numerics import NotPositiveDefinite, cholesky, cond1, logdet_from_chol, mahalanobis_sq


class SingularCandidate(Exception):
    pass


@dataclass
class CStepResult:
    H: np.ndarray              # sorted row positions of the converged h-subset
    mu: np.ndarray
    Sigma: np.ndarray          # unscaled covariance of H (denominator h-1)
    logdet: float              # log det Sigma
    steps: int                 # distance passes performed
    converged: bool
    logdets: list = field(default_factory=list)   # log det after each C-step


def h_subset(d2: np.ndarray, h: int) -> np.ndarray:
    """Indices of the h smallest d2, ties broken by index (R11); returned sorted."""
    idx = np.arange(d2.size)
    order = np.lexsort((idx, d2))
    return np.sort(order[:h])


def mean_cov(Z: np.ndarray, H: np.ndarray):
    """eqs. cstep4a/cstep4b."""
    ZH = Z[H]
    mu = ZH.mean(axis=0)
    D = ZH - mu[None, :]
    return mu, (D.T @ D) / (H.size - 1)


def concentrate(Z: np.ndarray, mu0: np.ndarray, Sigma0: np.ndarray, h: int,
                kappa_max: float = 1000.0, max_steps: int = 100) -> CStepResult:
    mu, Sigma = np.asarray(mu0, float), np.asarray(Sigma0, float)
    H = None
    logdets = []
    for step in range(1, max_steps + 1):
        try:
            cholesky(Sigma)
        except NotPositiveDefinite:
            raise SingularCandidate("Sigma_old not positive definite") from None
        if cond1(Sigma) >= kappa_max:
            raise SingularCandidate("condition number >= kappa_max")
        d2 = mahalanobis_sq(Z, mu, Sigma)
        Hn = h_subset(d2, h)
        if H is not None and np.array_equal(Hn, H):
            L = cholesky(Sigma)
            return CStepResult(H=H, mu=mu, Sigma=Sigma, logdet=logdet_from_chol(L),
                               steps=step, converged=True, logdets=logdets)
        H = Hn
        mu, Sigma = mean_cov(Z, H)
        try:
            logdets.append(logdet_from_chol(cholesky(Sigma)))
        except NotPositiveDefinite:
            raise SingularCandidate("h-subset covariance singular") from None
    L = cholesky(Sigma)
    return CStepResult(H=H, mu=mu, Sigma=Sigma, logdet=logdet_from_chol(L),
                       steps=max_steps, converged=False, logdets=logdets)


def delta_update(Z: np.ndarray, H_old: np.ndarray, H_new: np.ndarray,
                 mu_old: np.ndarray, Lambda_old: np.ndarray):
    """The paper's sequential update loop, leavers first.

    For each i with delta_i != 0: h <- h + delta_i; u = z_i - mu;
    mu <- mu + (delta_i / h) u; v = z_i - mu; Lambda <- Lambda + delta_i u v^T.
    Returns (mu_new, Lambda_new).
    """
    old = np.zeros(Z.shape[0], dtype=np.int64)
    new = np.zeros(Z.shape[0], dtype=np.int64)
    old[H_old] = 1
    new[H_new] = 1
    delta = new - old
    h = int(old.sum())
    mu = mu_old.copy()
    Lam = Lambda_old.copy()
    order = list(np.nonzero(delta < 0)[0]) + list(np.nonzero(delta > 0)[0])
    for i in order:
        d = int(delta[i])
        h += d
        u = Z[i] - mu
        mu = mu + (d / h) * u
        v = Z[i] - mu
        Lam = Lam + d * np.outer(u, v)
    return mu, Lam
