"""Chi-square quantiles and the MCD consistency factor (oracle; test infrastructure only).

PAPER.md:213-216 (§2.1): cut-off c_p = sqrt(chi2_{p,0.975}).
PAPER.md:158-164 (§2.1): consistency factor c(alpha) of Croux & Haesbroeck,
formula not printed in the paper; reading R1:
    c(alpha, p) = alpha / F_{chi2_{p+2}}(chi2_{p,alpha}),  c(1, p) = 1.
Library primitives: scipy.special.gammainc (regularised incomplete gamma) and
scipy.special.gammaincinv (its inverse).  Pinned in tests/test_oracle_chi2.py
by closed forms (p = 1 via erf, p = 2 via exp/log, even p via Poisson sums).
"""
from __future__ import annotations

from scipy.special import gammainc, gammaincinv


def chi2_cdf(x: float, dof: int) -> float:
    """F_{chi2_dof}(x) = P(dof/2, x/2)."""
    if x <= 0.0:
        return 0.0
    return float(gammainc(0.5 * dof, 0.5 * x))


def chi2_quantile(prob: float, dof: int) -> float:
    """chi2_{dof, prob}: the x with F_{chi2_dof}(x) = prob."""
    if not (0.0 < prob < 1.0):
        raise ValueError("prob must lie in (0, 1)")
    return float(2.0 * gammaincinv(0.5 * dof, prob))


def consistency_factor(alpha: float, p: int) -> float:
    """c(alpha, p) = alpha / F_{chi2_{p+2}}(chi2_{p,alpha}) (reading R1); c(1, p) = 1."""
    if alpha >= 1.0:
        return 1.0
    return alpha / chi2_cdf(chi2_quantile(alpha, p), p + 2)
