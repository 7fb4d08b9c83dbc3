"""The two new initial estimators S~1 (wrapping) and S~2 (LR-GSSCM) (oracle; test infrastructure only).

PAPER.md:467-503 (§3.2, eq. wrapping): g(z) = z if |z| <= b;
    q1 tanh(q2 (c - |z|)) sign(z) if b < |z| <= c; 0 if |z| > c,
    b = 1.5, c = 4, q1 = 1.541, q2 = 0.862; S~1 = covariance matrix of the
    wrapped data (reading R5: centred at the wrapped mean, denominator n-1).
PAPER.md:517-537 (§3.2, eq. LR): S~2 = (1/n) sum_i xi^2(||z_i||) z_i z_i^T,
    xi(r) = 1 (r <= A), (B - r)/(B - A) (A < r <= B), 0 (r > B).
    Reading R6: A = median(||z_i||), B = A + 1.5 IQR(||z_i||), type-7
    quantiles; ||z_i|| accumulated over j = 0..p-1 in that order.
"""
from __future__ import annotations

import numpy as np

WRAP_B, WRAP_C, WRAP_Q1, WRAP_Q2 = 1.5, 4.0, 1.541, 0.862


class DegenerateNorms(Exception):
    pass


def wrap(z: np.ndarray) -> np.ndarray:
    """Wrapping transform g applied elementwise."""
    z = np.asarray(z, dtype=np.float64)
    az = np.abs(z)
    mid = WRAP_Q1 * np.tanh(WRAP_Q2 * (WRAP_C - az)) * np.sign(z)
    return np.where(az <= WRAP_B, z, np.where(az <= WRAP_C, mid, 0.0))


def wrapped_covariance(Z: np.ndarray) -> np.ndarray:
    """S~1: classical covariance of g(Z)."""
    W = wrap(Z)
    n = W.shape[0]
    Wc = W - W.mean(axis=0)[None, :]
    return (Wc.T @ Wc) / (n - 1)


def row_norms(Z: np.ndarray) -> np.ndarray:
    """||z_i||, summing z_ij^2 over j = 0..p-1 in order (no fused multiply-add)."""
    acc = np.zeros(Z.shape[0])
    for j in range(Z.shape[1]):
        col = Z[:, j]
        acc = acc + col * col
    return np.sqrt(acc)


def quantile7(sorted_r: np.ndarray, prob: float) -> float:
    """Type-7 quantile of an ascending sample: y[j] + g (y[j+1] - y[j]), h = (n-1) prob."""
    n = sorted_r.size
    hpos = (n - 1) * prob
    j = int(np.floor(hpos))
    g = hpos - j
    if j + 1 >= n:
        return float(sorted_r[n - 1])
    return float(sorted_r[j] + g * (sorted_r[j + 1] - sorted_r[j]))


def lr_cutoffs(r: np.ndarray):
    """(A, B) = (median, median + 1.5 IQR) of the norms (reading R6)."""
    s = np.sort(r)
    A = quantile7(s, 0.5)
    iqr = quantile7(s, 0.75) - quantile7(s, 0.25)
    if not iqr > 0.0:
        raise DegenerateNorms("IQR of the norms is zero")
    return A, A + 1.5 * iqr


def xi(r: np.ndarray, A: float, B: float) -> np.ndarray:
    """Linearly redescending weight xi(r)."""
    return np.where(r <= A, 1.0, np.where(r <= B, (B - r) / (B - A), 0.0))


def gsscm_lr(Z: np.ndarray) -> np.ndarray:
    """S~2 = (1/n) sum xi^2(||z_i||) z_i z_i^T; z not re-centred."""
    r = row_norms(Z)
    A, B = lr_cutoffs(r)
    w = xi(r, A, B)
    Zw = Z * w[:, None]
    return (Zw.T @ Zw) / Z.shape[0]
