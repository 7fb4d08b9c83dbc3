"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no MCD, no C-step, no
estimator): it only draws data matrices with the shapes, covariance structure
and contamination families of BASELINE.json `configs` (which reuse the
paper's §5 families: shift / cluster / point contamination).
Both the oracle and the CUDA path consume its output byte-identically.

Recipe:
  * Sigma: Haar-random orthogonal Q (QR of a Gaussian matrix, sign-fixed),
    eigenvalues r^{(j-1)/(p-1)}, S = Q diag(lam) Q^T rescaled to unit diagonal;
    r is bisected (same Q) until kappa_2(Sigma) equals the target condition
    number (100; 50 for config 5).
  * inliers x = L g, L = chol(Sigma), g ~ N(0, I).
  * outlier rows: the first floor(eps n) entries of a seeded permutation.
  * shift by Mahalanobis distance d along v_min: x += d sqrt(lam_min) v_min.
  * cluster: m = d u / sqrt(u^T Sigma^-1 u), u uniform on the sphere; x = m + s L g.
  * sphere: x = R L g / ||g||.
  * config 5: y = L g, y_i += 7 u_i / sqrt(u_i^T Sigma^-1 u_i) on 2% rows, x = exp(y).
Generator: numpy PCG64 via default_rng([191005615, cfg(, batch)]).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_BASE = 191005615


@dataclass
class Dataset:
    X: np.ndarray                 # n x p, float64, C-contiguous (row = observation)
    h: int
    q: int
    log_transform: bool
    sigma: np.ndarray             # generating Sigma (log scale for config 5)
    outliers: np.ndarray          # bool mask of contaminated rows
    name: str
    meta: dict = field(default_factory=dict)


def random_correlation(rng: np.random.Generator, p: int, kappa: float) -> np.ndarray:
    """Random correlation matrix with 2-norm condition number `kappa` (bisection on r)."""
    if p == 1:
        return np.ones((1, 1))
    G = rng.standard_normal((p, p))
    Q, R = np.linalg.qr(G)
    Q = Q * np.sign(np.diag(R))

    def build(logr):
        lam = np.exp(logr * np.arange(p) / (p - 1))
        S = (Q * lam) @ Q.T
        d = 1.0 / np.sqrt(np.diag(S))
        S = S * d[:, None] * d[None, :]
        return 0.5 * (S + S.T)

    def cond(S):
        w = np.linalg.eigvalsh(S)
        return w[-1] / w[0]

    lo, hi = 0.0, -1.0
    while cond(build(hi)) < kappa:
        hi *= 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if cond(build(mid)) < kappa:
            lo = mid
        else:
            hi = mid
        if abs(hi - lo) < 1e-15:
            break
    return build(0.5 * (lo + hi))


def _gauss_rows(rng, n, L, chunk=1 << 20):
    p = L.shape[0]
    out = np.empty((n, p))
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        out[s:e] = rng.standard_normal((e - s, p)) @ L.T
    return out


def _mahal_unit(rng, Sigma, k):
    """k directions u_i/sqrt(u_i^T Sigma^-1 u_i) (Mahalanobis length 1)."""
    p = Sigma.shape[0]
    U = rng.standard_normal((k, p))
    U /= np.linalg.norm(U, axis=1, keepdims=True)
    Si = np.linalg.inv(Sigma)
    md = np.sqrt(np.einsum("ij,jk,ik->i", U, Si, U))
    return U / md[:, None]


def _vmin(Sigma):
    w, V = np.linalg.eigh(Sigma)
    v = V[:, 0]
    if v[np.argmax(np.abs(v))] < 0:
        v = -v
    return w[0], v


def make_config(cfg: int, n: int | None = None, batch: int | None = None) -> Dataset:
    """BASELINE.json configs[cfg-1]; `n` overrides the row count (same recipe)."""
    key = [SEED_BASE, cfg] if batch is None else [SEED_BASE, cfg, batch]
    if cfg == 1:
        N, p = 1000, 5
        n = n or N
        rng = np.random.default_rng(key)
        Sigma = random_correlation(rng, p, 100.0)
        L = np.linalg.cholesky(Sigma)
        X = _gauss_rows(rng, n, L)
        k = int(math.floor(0.10 * n))
        out_idx = rng.permutation(n)[:k]
        lam, v = _vmin(Sigma)
        X[out_idx] += 10.0 * math.sqrt(lam) * v
        h = int(math.floor(0.75 * n)); q = 1; log = False
    elif cfg == 2:
        N, p = 100_000, 10
        n = n or N
        rng = np.random.default_rng(key)
        Sigma = random_correlation(rng, p, 100.0)
        L = np.linalg.cholesky(Sigma)
        X = _gauss_rows(rng, n, L)
        k = int(math.floor(0.20 * n))
        out_idx = rng.permutation(n)[:k]
        m = 6.0 * _mahal_unit(rng, Sigma, 1)[0]
        X[out_idx] = m + 0.01 * (rng.standard_normal((k, p)) @ L.T)
        h = int(math.floor(0.75 * n)); q = 1; log = False
    elif cfg == 3:
        N, p = 1_000_000, 20
        n = n or N
        rng = np.random.default_rng(key)
        Sigma = random_correlation(rng, p, 100.0)
        L = np.linalg.cholesky(Sigma)
        X = _gauss_rows(rng, n, L)
        k = int(math.floor(0.20 * n))
        out_idx = rng.permutation(n)[:k]
        from scipy.stats import chi2  # radius constant only (BASELINE.json configs[2])
        R = 2.0 * math.sqrt(chi2.ppf(0.999, p))
        G = rng.standard_normal((k, p))
        G /= np.linalg.norm(G, axis=1, keepdims=True)
        X[out_idx] = R * (G @ L.T)
        h = int(math.floor(0.5 * n)) + 1; q = 1; log = False
    elif cfg == 4:
        N, p = 8_000_000, 40
        n = n or N
        rng = np.random.default_rng(key)
        Sigma = random_correlation(rng, p, 100.0)
        L = np.linalg.cholesky(Sigma)
        X = _gauss_rows(rng, n, L)
        k = int(math.floor(0.10 * n))
        perm = rng.permutation(n)[:k]
        ks = k // 2
        sh_idx, cl_idx = perm[:ks], perm[ks:]
        lam, v = _vmin(Sigma)
        X[sh_idx] += 8.0 * math.sqrt(lam) * v
        m = 8.0 * _mahal_unit(rng, Sigma, 1)[0]
        X[cl_idx] = m + 0.05 * (rng.standard_normal((len(cl_idx), p)) @ L.T)
        out_idx = perm
        kinds = {"shift_rows": np.sort(sh_idx), "cluster_rows": np.sort(cl_idx)}
        h = int(math.floor(0.75 * n)); q = 8; log = False
    elif cfg == 5:
        N, p = 20_000, 8
        n = n or N
        rng_s = np.random.default_rng([SEED_BASE, 5])
        Sigma = random_correlation(rng_s, p, 50.0)
        L = np.linalg.cholesky(Sigma)
        rng = np.random.default_rng([SEED_BASE, 5, 0 if batch is None else batch])
        Y = _gauss_rows(rng, n, L)
        k = int(math.floor(0.02 * n))
        out_idx = rng.permutation(n)[:k]
        Y[out_idx] += 7.0 * _mahal_unit(rng, Sigma, k)
        X = np.exp(Y)
        h = int(math.floor(0.75 * n)); q = 1; log = True
    else:
        raise ValueError(f"unknown config {cfg}")
    mask = np.zeros(n, dtype=bool)
    mask[out_idx] = True
    meta = {"n": n, "p": X.shape[1]}
    if cfg == 4:
        meta.update(kinds)
    return Dataset(X=np.ascontiguousarray(X), h=h, q=q, log_transform=log, sigma=Sigma,
                   outliers=mask, name=f"cfg{cfg}", meta=meta)


def gaussian(n: int, p: int, seed: int, sigma: np.ndarray | None = None) -> np.ndarray:
    """Plain N(0, Sigma) rows (used by small property tests)."""
    rng = np.random.default_rng([SEED_BASE, 1000, seed])
    if sigma is None:
        return rng.standard_normal((n, p))
    return rng.standard_normal((n, p)) @ np.linalg.cholesky(sigma).T


def a09(p: int) -> np.ndarray:
    """A09 scatter Sigma_jk = (-0.9)^|j-k|."""
    j = np.arange(p)
    return (-0.9) ** np.abs(j[:, None] - j[None, :])


def paper_simulation(p: int, eps: float, kind: str, rep: int, n: int = 65536, gamma: float = 50.0) -> Dataset:
    """The paper's simulation design (Table 2): n cases from N(0, Sigma) with the
    A09 Sigma, floor(eps n) random cases replaced by outliers around mu_C = gamma v, v the last
    eigenvector of Sigma rescaled to v^T Sigma^-1 v = p:
      point   -- every outlier at mu_C;
      shift   -- N(mu_C, Sigma);
      cluster -- N(mu_C, 0.05^2 I).
    Seeded by default_rng([191005615, 2000, p, round(1000 eps), kind index, rep])."""
    kinds = ("point", "shift", "cluster")
    rng = np.random.default_rng([SEED_BASE, 2000, p, int(round(1000 * eps)), kinds.index(kind), rep])
    Sigma = a09(p)
    L = np.linalg.cholesky(Sigma)
    X = rng.standard_normal((n, p)) @ L.T
    w, V = np.linalg.eigh(Sigma)
    v = V[:, 0]                                   # eigenvector of the smallest eigenvalue
    v = v * math.sqrt(p / (v @ np.linalg.solve(Sigma, v)))
    mu_c = gamma * v
    k = int(math.floor(eps * n))
    idx = rng.choice(n, size=k, replace=False)
    if kind == "point":
        X[idx] = mu_c
    elif kind == "shift":
        X[idx] = mu_c + rng.standard_normal((k, p)) @ L.T
    else:
        X[idx] = mu_c + 0.05 * rng.standard_normal((k, p))
    mask = np.zeros(n, dtype=bool)
    mask[idx] = True
    return Dataset(X=np.ascontiguousarray(X), h=n // 2, q=1, log_transform=False, sigma=Sigma, outliers=mask,
                   name=f"sim_a09_p{p}_{kind}_{eps}", meta={"n": n, "p": p, "gamma": gamma, "rep": rep})
