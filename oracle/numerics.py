"""Small dense linear algebra for p <= 40 (oracle; test infrastructure only).

PAPER.md:617-641 (§3.4): Sigma = L L^T, det(Sigma) = (prod L_jj)^2.
PAPER.md:643-657 (§3.4): condition monitor ||Sigma||_1 ||Sigma^-1||_1 >= kappa_max.
PAPER.md:559-573 (§3.3 step 1): S = V D V^T with decreasing eigenvalues.
Library primitives used as single steps: numpy.linalg.cholesky / inv / eigh.
"""
from __future__ import annotations

import numpy as np


class NotPositiveDefinite(Exception):
    pass


def cholesky(S: np.ndarray) -> np.ndarray:
    """Lower-triangular L with L L^T = S; raises NotPositiveDefinite."""
    try:
        L = np.linalg.cholesky(S)
    except np.linalg.LinAlgError as e:
        raise NotPositiveDefinite(str(e)) from None
    if not np.all(np.isfinite(L)) or np.any(np.diag(L) <= 0.0):
        raise NotPositiveDefinite("non-positive pivot")
    return L


def logdet_from_chol(L: np.ndarray) -> float:
    """log det(Sigma) = 2 sum_j log L_jj."""
    return float(2.0 * np.sum(np.log(np.diag(L))))


def cond1(S: np.ndarray) -> float:
    """||S||_1 ||S^-1||_1 with the exact inverse."""
    Si = np.linalg.inv(S)
    return float(np.max(np.sum(np.abs(S), axis=0)) * np.max(np.sum(np.abs(Si), axis=0)))


def eigh_desc(S: np.ndarray):
    """Eigenpairs of symmetric S, eigenvalues descending.

    Sign convention (immaterial for Sigma_k = V D~ V^T, reading R9): the
    component of largest magnitude of each eigenvector is made positive.
    """
    w, V = np.linalg.eigh(0.5 * (S + S.T))
    order = np.argsort(-w, kind="stable")
    w = w[order]
    V = V[:, order].copy()
    for j in range(V.shape[1]):
        k = int(np.argmax(np.abs(V[:, j])))
        if V[k, j] < 0:
            V[:, j] = -V[:, j]
    return w, V


def mahalanobis_sq(Z: np.ndarray, mu: np.ndarray, Sigma: np.ndarray) -> np.ndarray:
    """d^2(z_i, mu, Sigma) = (z_i - mu)^T Sigma^-1 (z_i - mu), plain definition."""
    D = Z - mu[None, :]
    Y = np.linalg.solve(Sigma, D.T).T
    return np.einsum("ij,ij->i", D, Y)
