"""The whole RT-DetMCD fit and the flag pass (oracle; test infrastructure only).

Serial RT-DetMCD (variant IDC) and parallel IDCP_q
(Figs. 2-3), written step by step in the paper's order:
  1. standardise every column with the univariate reweighted MCD over all n
     rows (global estimates for the blocks);
  2. (q > 1) random partition into q blocks of m = floor(n/q);
  3. per block: S~1, S~2 -> refinement
     -> C-steps to convergence -> c(alpha)-scaled candidates;
     the raw block fit is the candidate with the lower determinant
     (ties -> start 1);
  4. (q > 1) entrywise median, KL ranking, ceil(q/2) kept, pooled;
  5. reweighting: mean and covariance of the rows whose RD does not exceed
     c_p = sqrt(chi2_{p,0.975}) (distributed version
     PAPER.md:975-995 = the same union, reading R16), scaled by c(0.975, p)
     (reading R17);
  6. flag rows whose final RD exceeds c_p, all n rows.
Outputs are reported in standardized units and de-standardized to X units
(mu_X = loc + scale * mu_Z, Sigma_X = diag(scale) Sigma_Z diag(scale)).
Readings R18: block coverage h_l = floor(h m / n); alpha_l = h_l / m.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .chi2 import chi2_quantile, consistency_factor
from .cstep import SingularCandidate, concentrate
from .initial import DegenerateNorms, gsscm_lr, wrapped_covariance
from .numerics import NotPositiveDefinite, cholesky, logdet_from_chol, mahalanobis_sq
from .parallel import block_rows, partition, select_and_pool
from .refine import IllConditioned, refine
from .unimcd import DegenerateScale, unimcd_reweighted


class FitError(Exception):
    def __init__(self, code: str, msg: str):
        super().__init__(f"{code}: {msg}")
        self.code = code


@dataclass
class StartResult:
    ok: bool
    reason: str = ""
    mu0: np.ndarray | None = None        # refined start
    Sigma0: np.ndarray | None = None
    H: np.ndarray | None = None
    mu: np.ndarray | None = None
    Sigma: np.ndarray | None = None      # unscaled h-subset covariance
    logdet: float = math.inf
    steps: int = 0
    converged: bool = False
    logdets: list = field(default_factory=list)


@dataclass
class BlockFit:
    block: int
    rows: np.ndarray                     # original row indices, by position in block
    m: int
    h: int
    starts: list
    chosen: int                          # 0 = wrapping start, 1 = GSSCM start, -1 failed
    mu: np.ndarray | None = None
    Sigma_raw: np.ndarray | None = None  # c(alpha_l) * unscaled
    logdet: float = math.inf


@dataclass
class FitResult:
    n: int
    p: int
    h: int
    q: int
    loc: np.ndarray
    scale: np.ndarray
    blocks: list
    mu_raw_z: np.ndarray
    Sigma_raw_z: np.ndarray
    kept_blocks: list
    weights: np.ndarray                  # bool, n (False for the partition remainder)
    mu_rew_z: np.ndarray
    Sigma_rew_z: np.ndarray
    rd2: np.ndarray                      # final squared robust distances, n
    flags: np.ndarray                    # bool, n
    cutoff2: float
    mu_raw: np.ndarray
    Sigma_raw: np.ndarray
    mu_rew: np.ndarray
    Sigma_rew: np.ndarray
    warnings: list


def standardize(X: np.ndarray):
    """(loc_j, scale_j) = univariate reweighted MCD of column j."""
    p = X.shape[1]
    loc = np.empty(p)
    scale = np.empty(p)
    for j in range(p):
        try:
            u = unimcd_reweighted(X[:, j])
        except DegenerateScale:
            raise FitError("DEGENERATE_COLUMN", f"column {j}") from None
        loc[j], scale[j] = u.loc, u.scale
    return loc, scale


def run_start(Zb: np.ndarray, S: np.ndarray, hb: int, kappa_max: float, max_csteps: int) -> StartResult:
    try:
        ref = refine(S, Zb, kappa_max)
    except (IllConditioned, DegenerateScale) as e:
        return StartResult(ok=False, reason=f"refine: {e}")
    try:
        c = concentrate(Zb, ref.mu, ref.Sigma, hb, kappa_max, max_csteps)
    except (SingularCandidate, NotPositiveDefinite) as e:
        return StartResult(ok=False, reason=f"cstep: {e}", mu0=ref.mu, Sigma0=ref.Sigma)
    return StartResult(ok=True, mu0=ref.mu, Sigma0=ref.Sigma, H=c.H, mu=c.mu, Sigma=c.Sigma,
                       logdet=c.logdet, steps=c.steps, converged=c.converged, logdets=c.logdets)


def fit_block(Zb: np.ndarray, hb: int, kappa_max: float = 1000.0, max_csteps: int = 100):
    """Steps 1-4 of PAPER.md:811-840 for one block; returns (starts, chosen)."""
    starts = []
    S1 = wrapped_covariance(Zb)
    starts.append(run_start(Zb, S1, hb, kappa_max, max_csteps))
    try:
        S2 = gsscm_lr(Zb)
        starts.append(run_start(Zb, S2, hb, kappa_max, max_csteps))
    except DegenerateNorms as e:
        starts.append(StartResult(ok=False, reason=f"S2: {e}"))
    ok = [k for k in range(2) if starts[k].ok]
    if not ok:
        return starts, -1
    chosen = ok[0]
    if len(ok) == 2 and starts[1].logdet < starts[0].logdet:
        chosen = 1
    return starts, chosen


def warm_block(Zb: np.ndarray, mu0: np.ndarray, Sigma0: np.ndarray, hb: int, kappa_max: float = 1000.0,
               max_csteps: int = 100):
    """Warm start (§4 closing note): the previous run's reweighted estimate,
    expressed in this run's standardised units, is the input of step 3 -- the C-steps of
    PAPER.md:822-827 -- of every block; steps 1-2 (initial estimators, refinement) are skipped.
    Reading W1: a warm start the C-step cannot take (not PD, condition >= kappa_max) fails the
    block like a dropped start (reading R10).  Returns (starts, chosen) like fit_block."""
    try:
        c = concentrate(Zb, mu0, Sigma0, hb, kappa_max, max_csteps)
    except (SingularCandidate, NotPositiveDefinite) as e:
        return [StartResult(ok=False, reason=f"warm: {e}", mu0=mu0, Sigma0=Sigma0)], -1
    st = StartResult(ok=True, mu0=mu0, Sigma0=Sigma0, H=c.H, mu=c.mu, Sigma=c.Sigma, logdet=c.logdet,
                     steps=c.steps, converged=c.converged, logdets=c.logdets)
    return [st], 0


def fit(X: np.ndarray, h: int | None = None, alpha: float = 0.5, q: int = 1, seed: int = 0,
        kappa_max: float = 1000.0, quantile: float = 0.975, max_csteps: int = 100,
        log_transform: bool = False, partition_mode: str = "permute", warm_start=None,
        consistency: str = "alpha") -> FitResult:
    """warm_start: optional (mu, Sigma) of a previous fit in the units this fit reports (after ln
    when log_transform) -- the single C-step start of every block (warm_block).

    consistency: "alpha" -- Sigma_raw = c(alpha) Sigma_H, the factor the text defines (PAPER.md:158-175,
    reading R1); "median" -- Sigma_raw = median_i d^2(z_i; mu_H, Sigma_H) / chi2_{p,0.5} Sigma_H over the
    rows of the block, the rule that reproduces the paper's Table 2 (DESIGN.md finding F1)."""
    if consistency not in ("alpha", "median"):
        raise FitError("INVALID_ARG", f"consistency {consistency}")
    X = np.asarray(X, dtype=np.float64)
    n, p = X.shape
    if not np.all(np.isfinite(X)):
        raise FitError("NONFINITE", f"row {int(np.nonzero(~np.isfinite(X).all(1))[0][0])}")
    if log_transform:
        if np.any(X <= 0):
            raise FitError("INVALID_ARG", "log transform needs positive data")
        X = np.log(X)
    if h is None or h == 0:
        h = int(math.floor(alpha * n))
    if not (n > 2 * p and p < h <= n and q >= 1):
        raise FitError("INVALID_ARG", f"n={n} p={p} h={h} q={q}")
    warnings = []
    if h < (n + p + 1) // 2:
        warnings.append("H_BELOW_BOUND")
    loc, scale = standardize(X)
    Z = (X - loc[None, :]) / scale[None, :]
    block, pos, m = partition(n, q, seed, partition_mode)
    hb = (h * m) // n
    if not hb > p:
        raise FitError("INVALID_ARG", "block h_l <= p")
    blocks = []
    for l in range(q):
        rows = block_rows(block, pos, l, m)
        Zb = Z[rows]
        if warm_start is None:
            starts, chosen = fit_block(Zb, hb, kappa_max, max_csteps)
        else:
            mu_w = (np.asarray(warm_start[0], float) - loc) / scale
            S_w = np.asarray(warm_start[1], float) / np.outer(scale, scale)
            starts, chosen = warm_block(Zb, mu_w, S_w, hb, kappa_max, max_csteps)
        bf = BlockFit(block=l, rows=rows, m=m, h=hb, starts=starts, chosen=chosen)
        if chosen >= 0:
            st = starts[chosen]
            bf.mu = st.mu
            if consistency == "median":
                factor = float(np.median(mahalanobis_sq(Zb, st.mu, st.Sigma))) / chi2_quantile(0.5, p)
            else:
                factor = consistency_factor(hb / m, p)
            bf.Sigma_raw = factor * st.Sigma
            bf.logdet = st.logdet
            if not st.converged:
                warnings.append(f"MAX_CSTEPS_BLOCK{l}")
        else:
            warnings.append(f"BLOCK_FAILED{l}")
        blocks.append(bf)
    valid = [b for b in blocks if b.chosen >= 0]
    if q == 1:
        if not valid:
            raise FitError("BOTH_STARTS_FAILED", "both starts failed")
        mu_raw, Sigma_raw, kept = valid[0].mu, valid[0].Sigma_raw, [0]
    else:
        if len(valid) < q - q // 2:
            raise FitError("TOO_FEW_VALID_BLOCKS", f"{len(valid)} of {q} valid")
        mu_raw, Sigma_raw, kept, _ = select_and_pool([b.mu for b in valid], [b.Sigma_raw for b in valid],
                                                     [b.m for b in valid], [b.block for b in valid])
    # reweighting over the fitted rows
    fitted = block >= 0
    c2 = chi2_quantile(quantile, p)
    try:
        cholesky(Sigma_raw)
    except NotPositiveDefinite:
        raise FitError("NOT_PD", "raw scatter not positive definite") from None
    d2_raw = mahalanobis_sq(Z, mu_raw, Sigma_raw)
    weights = fitted & (d2_raw <= c2)
    k = int(weights.sum())
    if k <= p:
        raise FitError("NOT_PD", "too few reweighted inliers")
    Zw = Z[weights]
    mu_rew = Zw.mean(axis=0)
    D = Zw - mu_rew[None, :]
    Sigma_rew = consistency_factor(quantile, p) * (D.T @ D) / (k - 1)
    try:
        cholesky(Sigma_rew)
    except NotPositiveDefinite:
        raise FitError("NOT_PD", "reweighted scatter not positive definite") from None
    rd2 = mahalanobis_sq(Z, mu_rew, Sigma_rew)
    flags = rd2 > c2
    ss = np.outer(scale, scale)
    return FitResult(n=n, p=p, h=h, q=q, loc=loc, scale=scale, blocks=blocks,
                     mu_raw_z=mu_raw, Sigma_raw_z=Sigma_raw, kept_blocks=kept,
                     weights=weights, mu_rew_z=mu_rew, Sigma_rew_z=Sigma_rew,
                     rd2=rd2, flags=flags, cutoff2=c2,
                     mu_raw=loc + scale * mu_raw, Sigma_raw=Sigma_raw * ss,
                     mu_rew=loc + scale * mu_rew, Sigma_rew=Sigma_rew * ss,
                     warnings=warnings)


def flag(X: np.ndarray, mu: np.ndarray, Sigma: np.ndarray, quantile: float = 0.975):
    """Step 10 / rtdetmcd_flag: RD^2 under (mu, Sigma) in X units and flags RD^2 > chi2_{p,q}."""
    X = np.asarray(X, dtype=np.float64)
    c2 = chi2_quantile(quantile, X.shape[1])
    rd2 = mahalanobis_sq(X, np.asarray(mu, float), np.asarray(Sigma, float))
    return rd2, rd2 > c2, c2


def logdet(S: np.ndarray) -> float:
    return logdet_from_chol(cholesky(S))
