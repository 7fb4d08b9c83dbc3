"""Refinement of an initial scatter estimate (oracle; test infrastructure only).

PAPER.md:559-605 (§3.3, steps 1-4):
  1. S~_k = V D V^T, eigenvalues decreasing; scores T = Z V.
  2. if lambda_1/lambda_p exceeds kappa_max (=1000) the start is dropped
     (reading R7: also dropped when lambda_p <= 0; comparator '>').
  3. D~ = diag(sigma_uni^2(T_1), ..., sigma_uni^2(T_p)); Sigma_k = V D~ V^T.
  4. Z~ = Z Sigma_k^{-1/2} (row-wise sphering); mu_k = Sigma_k^{1/2} (mu_uni(Z~_j))_j.
Reading R8: "univariate MCD" = the reweighted univariate MCD of §3.1.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .numerics import eigh_desc
from .unimcd import unimcd_reweighted


class IllConditioned(Exception):
    pass


@dataclass
class Refined:
    mu: np.ndarray
    Sigma: np.ndarray
    V: np.ndarray
    lam: np.ndarray          # eigenvalues of the initial estimate
    dtilde: np.ndarray       # robust eigenvalues D~
    mutilde: np.ndarray      # univariate locations of the sphered columns


def refine(S: np.ndarray, Z: np.ndarray, kappa_max: float = 1000.0) -> Refined:
    lam, V = eigh_desc(S)
    if not lam[-1] > 0.0 or lam[0] / lam[-1] > kappa_max:
        raise IllConditioned(f"lambda_1/lambda_p = {lam[0] / lam[-1] if lam[-1] > 0 else np.inf}")
    T = Z @ V
    p = Z.shape[1]
    dt = np.array([unimcd_reweighted(T[:, j]).scale ** 2 for j in range(p)])
    Sigma = (V * dt) @ V.T
    Sig_mhalf = (V * (1.0 / np.sqrt(dt))) @ V.T
    Sig_half = (V * np.sqrt(dt)) @ V.T
    Zt = Z @ Sig_mhalf
    mt = np.array([unimcd_reweighted(Zt[:, j]).loc for j in range(p)])
    mu = Sig_half @ mt
    return Refined(mu=mu, Sigma=Sigma, V=V, lam=lam, dtilde=dt, mutilde=mt)
