"""Univariate raw and reweighted MCD (oracle; test infrastructure only).

PAPER.md:432-453 (§3.1): "we now use the univariate reweighted MCD estimator
... with coverage h~ = [n/2]+1.  ... for univariate data, the raw MCD
estimates reduce to the mean and the standard deviation of the h~-subset with
smallest variance.  They can be computed in O(n log(n)) time ... by sorting
the data, followed by looping over contiguous h~-subsets".

Readings:
  R2  objective SQ(s) = sum_{i=s}^{s+h-1} (y_(i) - ybar_s)^2 over the sorted
      sample; s* = argmin, ties -> lowest s.  The argmin is the EXACT one for
      the given fp64 values: an fp64 sliding pass shortlists every s whose
      value lies within a rigorous rounding bound of the minimum, and those
      are re-evaluated in exact integer arithmetic (h SQ(s) = h S2 - S1^2).
  R3  raw location = window mean; raw variance = c(h/n, 1) SQ(s*)/(h-1).
  R4  reweighting keeps x with (x - loc0)^2 <= chi2_{1,0.975} * var0 (fp64,
      that expression); loc = mean of kept (correctly rounded sum / k);
      scale^2 = c(0.975, 1) * sum_kept (x - loc)^2 / (k - 1).
Pinned by brute force over all C(n, h) subsets (n <= 12), SPEC examples and
exact power-of-two equivariance (tests/test_oracle_unimcd.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from .chi2 import chi2_quantile, consistency_factor

U = 2.0 ** -53


class DegenerateScale(Exception):
    pass


@dataclass
class UniRaw:
    start: int        # s* in the sorted sample
    loc: float        # window mean
    var_raw: float    # SQ(s*)/(h-1), no consistency factor
    var: float        # c(h/n,1) * var_raw


@dataclass
class UniMCD:
    loc: float
    scale: float
    raw: UniRaw
    n_kept: int


def _exact_ints(vals: np.ndarray):
    """vals_i = K_i * 2**E exactly, K_i Python ints."""
    m, e = np.frexp(vals)
    M = (m * 2.0 ** 53).astype(np.int64)          # exact 53-bit signed mantissas
    nz = M != 0
    E = (int(e[nz].min()) - 53) if nz.any() else 0
    sh = np.where(nz, e - 53 - E, 0).astype(np.int64)
    K = [int(a) << int(b) for a, b in zip(M.tolist(), sh.tolist())]
    return K, E


def _gamma(k: int) -> float:
    return k * U / (1.0 - k * U)


def unimcd_raw(x: np.ndarray, h: int) -> UniRaw:
    """Raw univariate MCD with coverage h, exact window argmin (R2)."""
    y = np.sort(np.asarray(x, dtype=np.float64), kind="stable")
    n = y.size
    if not (1 <= h <= n):
        raise ValueError("need 1 <= h <= n")
    ns = n - h + 1
    # --- fp64 screening pass (shifted by the middle order statistic) ---
    c = y[n // 2]
    a = y - c
    P1 = np.concatenate(([0.0], np.cumsum(a)))
    P2 = np.concatenate(([0.0], np.cumsum(a * a)))
    S1 = P1[h:h + ns] - P1[:ns]
    S2 = P2[h:h + ns] - P2[:ns]
    SQh = h * S2 - S1 * S1
    # rigorous bound on |computed - exact| of h*SQ(s) (x2 safety)
    A1 = float(np.sum(np.abs(a))) * (1 + U)
    A2 = float(np.sum(a * a)) * (1 + 4 * U)
    e1 = 2 * _gamma(n + 2) * A1 + U * np.abs(S1)
    e2 = 2 * _gamma(n + 4) * A2 + U * np.abs(S2)
    err = h * e2 + U * h * np.abs(S2) + 2 * np.abs(S1) * e1 + e1 * e1 + U * S1 * S1 + U * np.abs(SQh)
    err = 2.0 * err + 1e-300
    thresh = float(np.min(SQh + err))
    cand = np.nonzero(SQh - err <= thresh)[0]
    smin, smax = int(cand[0]), int(cand[-1])
    # --- exact evaluation over [smin, smax] by sliding integer sums ---
    K, E = _exact_ints(y[smin:smax + h])
    s1 = sum(K[:h])
    s2 = sum(k * k for k in K[:h])
    best_v = h * s2 - s1 * s1
    best_s, best_s1 = smin, s1
    for s in range(smin + 1, smax + 1):
        old = K[s - 1 - smin]
        new = K[s + h - 1 - smin]
        s1 += new - old
        s2 += new * new - old * old
        v = h * s2 - s1 * s1
        if v < best_v:
            best_v, best_s, best_s1 = v, s, s1
    scale2 = Fraction(2) ** E if E >= 0 else Fraction(1, 2 ** (-E))
    loc = float(Fraction(best_s1, h) * scale2)
    SQ = Fraction(best_v, h) * scale2 * scale2
    var_raw = float(SQ / (h - 1)) if h > 1 else 0.0
    var = consistency_factor(h / n, 1) * var_raw
    return UniRaw(start=best_s, loc=loc, var_raw=var_raw, var=var)


def unimcd_reweighted(x: np.ndarray) -> UniMCD:
    """Univariate reweighted MCD with h~ = floor(n/2)+1 (readings R3, R4)."""
    x = np.asarray(x, dtype=np.float64)
    n = x.size
    if n < 2:
        raise ValueError("need n >= 2")
    h = n // 2 + 1
    raw = unimcd_raw(x, h)
    if not raw.var > 0.0:
        raise DegenerateScale("raw MCD window has zero variance")
    q1 = chi2_quantile(0.975, 1)
    d = x - raw.loc
    keep = (d * d) <= q1 * raw.var
    kept = x[keep]
    k = kept.size
    if k < 2:
        raise DegenerateScale("fewer than two points kept")
    loc = math.fsum(kept.tolist()) / k
    r = kept - loc
    var = consistency_factor(0.975, 1) * (math.fsum((r * r).tolist()) / (k - 1))
    if not var > 0.0:
        raise DegenerateScale("reweighted variance is zero")
    return UniMCD(loc=loc, scale=math.sqrt(var), raw=raw, n_kept=int(k))
