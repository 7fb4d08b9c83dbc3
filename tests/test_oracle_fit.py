"""Whole-fit pins for oracle/fit.py: exact MCD brute force, equivariance, flag rates."""
import itertools

import numpy as np
import pytest

from oracle import fit as F
from oracle.chi2 import consistency_factor
from oracle.unimcd import unimcd_reweighted
from paper_1910_05615_b200 import datagen


def _exact_mcd_logdet(X, h):
    best = np.inf
    for S in itertools.combinations(range(X.shape[0]), h):
        C = np.cov(X[list(S)], rowvar=False)
        s, ld = np.linalg.slogdet(C)
        if s > 0 and ld < best:
            best = ld
    return best


def _raw_logdet_unscaled(r):
    b = r.blocks[0]
    return b.starts[b.chosen].logdet


@pytest.mark.parametrize("seed", range(3))
def test_detmcd_objective_at_least_exact_mcd(seed):
    # north_star: n = 12, p = 2, brute force over all C(12, 7) = 792 subsets
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((12, 2)) @ np.array([[1.0, 0.4], [0.0, 0.7]])
    X[:2] += 6.0
    r = F.fit(X, h=7)
    Xz = (X - r.loc) / r.scale
    exact = _exact_mcd_logdet(Xz, 7)
    assert _raw_logdet_unscaled(r) >= exact - 1e-12


def test_detmcd_equals_exact_mcd_when_separated():
    # 9 tight inliers + 3 far points, h = 9 (C(12, 9) = 220 subsets)
    rng = np.random.default_rng(10)
    X = np.vstack([rng.standard_normal((9, 2)) * 0.5, [[40.0, 40.0], [-35.0, 50.0], [60.0, -45.0]]])
    r = F.fit(X, h=9)
    Xz = (X - r.loc) / r.scale
    assert _raw_logdet_unscaled(r) == pytest.approx(_exact_mcd_logdet(Xz, 9), abs=1e-12)
    assert set(r.blocks[0].starts[r.blocks[0].chosen].H.tolist()) == set(range(9))


def test_raw_scatter_and_destandardisation():
    d = datagen.make_config(1)
    r = F.fit(d.X, h=d.h)
    b = r.blocks[0]
    H = b.starts[b.chosen].H
    XH = d.X[H]
    # A1: mean of H; c(alpha)/(h-1) SSCP, alpha = h/n — in X units
    assert np.allclose(r.mu_raw, XH.mean(0), rtol=1e-12, atol=1e-13)
    assert np.allclose(r.Sigma_raw, consistency_factor(d.h / 1000, 5) * np.cov(XH, rowvar=False), rtol=1e-11)
    # the standardisation is the univariate reweighted MCD of each column
    for j in range(5):
        u = unimcd_reweighted(d.X[:, j])
        assert r.loc[j] == u.loc and r.scale[j] == u.scale


def test_power_of_two_column_scaling_exact():
    d = datagen.make_config(1)
    s = 2.0 ** np.array([3, -2, 0, 5, -7])
    r = F.fit(d.X, h=d.h)
    r2 = F.fit(d.X * s, h=d.h)
    assert np.array_equal(r.flags, r2.flags)
    assert np.array_equal(r.blocks[0].starts[0].H, r2.blocks[0].starts[0].H)
    assert np.array_equal(r2.mu_rew, r.mu_rew * s)
    assert np.array_equal(r2.Sigma_rew, r.Sigma_rew * np.outer(s, s))


def test_translation_equivariance():
    d = datagen.make_config(1)
    a = np.array([10.0, -3.5, 100.25, 0.5, 7.0])
    r = F.fit(d.X, h=d.h)
    r2 = F.fit(d.X + a, h=d.h)
    assert np.array_equal(r.flags, r2.flags)
    assert np.allclose(r2.mu_rew, r.mu_rew + a, rtol=1e-12, atol=1e-10)
    assert np.allclose(r2.Sigma_rew, r.Sigma_rew, rtol=1e-9)


def test_row_permutation_invariance():
    d = datagen.make_config(1)
    P = np.random.default_rng(3).permutation(1000)
    r = F.fit(d.X, h=d.h)
    r2 = F.fit(d.X[P], h=d.h)
    assert np.array_equal(r.flags[P], r2.flags)
    assert np.allclose(r2.Sigma_rew, r.Sigma_rew, rtol=1e-12)
    b, b2 = r.blocks[0], r2.blocks[0]
    assert set(P[b2.starts[b2.chosen].H].tolist()) == set(b.starts[b.chosen].H.tolist())


def test_clean_flag_rate_and_shift_outliers():
    X = datagen.gaussian(20_000, 4, seed=20, sigma=datagen.a09(4))
    r = F.fit(X, alpha=0.75)
    assert abs(r.flags.mean() - 0.025) < 0.01
    d = datagen.make_config(1)
    r1 = F.fit(d.X, h=d.h)
    assert r1.flags[d.outliers].all()


def test_h_equal_n_gives_classical_raw():
    X = datagen.gaussian(300, 3, seed=21)
    r = F.fit(X, h=300)
    assert np.allclose(r.mu_raw, X.mean(0), rtol=1e-12, atol=1e-14)
    assert np.allclose(r.Sigma_raw, np.cov(X, rowvar=False), rtol=1e-11)


def test_blocked_fit_q1_equals_serial_and_q4_runs():
    d = datagen.make_config(2, n=20_000)
    r1 = F.fit(d.X, h=d.h, q=1)
    r4 = F.fit(d.X, h=d.h, q=4, seed=5)
    assert len(r4.blocks) == 4 and len(r4.kept_blocks) == 2
    assert r4.weights.sum() > 0.5 * 20_000
    # both fits see the same cluster-dominated geometry: the q=4 aggregate is close
    assert np.linalg.norm(r4.Sigma_rew - r1.Sigma_rew) / np.linalg.norm(r1.Sigma_rew) < 0.2


def test_errors():
    X = datagen.gaussian(50, 3, seed=22)
    with pytest.raises(F.FitError):
        F.fit(X[:5], h=4)
    Y = X.copy(); Y[3, 1] = np.nan
    with pytest.raises(F.FitError) as e:
        F.fit(Y, h=30)
    assert e.value.code == "NONFINITE"
    Y = X.copy(); Y[:, 2] = 1.0
    with pytest.raises(F.FitError) as e:
        F.fit(Y, h=30)
    assert e.value.code == "DEGENERATE_COLUMN"


def test_config4_recipe_cluster_absorbed():
    """Config 4's tight cluster N(m, 0.05^2 Sigma), |m|_M = 8, ends up INSIDE the DetMCD h-subsets at
    p = 40, h = 0.75 n: the subset holding the cluster has a lower determinant than the clean subset
    reached by C-steps from the generating (0, Sigma) (the MCD keeps the lowest
    determinant), so flagging only the shift rows is the estimator's answer, not a defect."""
    from oracle.cstep import concentrate
    n = 40_000
    d = datagen.make_config(4, n=n)
    o = F.fit(d.X, h=int(0.75 * n), q=8, seed=191005615, partition_mode="contiguous")
    sh, cl = d.meta["shift_rows"], d.meta["cluster_rows"]
    assert o.flags[sh].mean() > 0.99 and o.flags[cl].mean() == 0.0
    b = o.blocks[0]
    st = b.starts[b.chosen]
    Zb = ((d.X - o.loc) / o.scale)[b.rows]
    clean = concentrate(Zb, -o.loc / o.scale, d.sigma / np.outer(o.scale, o.scale), b.h)
    assert not np.isin(b.rows[clean.H], cl).any()
    assert np.isin(b.rows[st.H], cl).mean() > 0.05
    assert st.logdet < clean.logdet - 1.0


def test_warm_start_from_cold_raw_fit_reproduces_it():
    """A warm start at the cold fit's own raw estimate: its h-subset is a C-step fixed point
     and a positive multiple of Sigma ranks distances identically, so the
    first C-step returns the same subset and the warm fit equals the cold fit exactly."""
    d = datagen.make_config(1)
    cold = F.fit(d.X, h=d.h)
    warm = F.fit(d.X, h=d.h, warm_start=(cold.mu_raw, cold.Sigma_raw))
    st_c = cold.blocks[0].starts[cold.blocks[0].chosen]
    st_w = warm.blocks[0].starts[0]
    assert np.array_equal(st_c.H, st_w.H) and st_w.steps == 2  # one C-step + the pass confirming H_new == H_old
    assert np.allclose(warm.Sigma_rew, cold.Sigma_rew, rtol=1e-13, atol=1e-15)
    assert np.array_equal(warm.flags, cold.flags)


def test_warm_start_stream_and_failure():
    """Config 5 stream: batch 1 warm-started from batch 0's reweighted fit flags the 2% shifted rows
    like the cold fit; a singular warm start fails the block (reading W1)."""
    b0, b1 = datagen.make_config(5, batch=0), datagen.make_config(5, batch=1)
    f0 = F.fit(b0.X, h=b0.h, log_transform=True)
    cold = F.fit(b1.X, h=b1.h, log_transform=True)
    warm = F.fit(b1.X, h=b1.h, log_transform=True, warm_start=(f0.mu_rew, f0.Sigma_rew))
    assert warm.flags[b1.outliers].mean() > 0.97
    assert (warm.flags == cold.flags).mean() > 0.995
    p = b1.X.shape[1]
    with pytest.raises(F.FitError) as e:
        F.fit(b1.X, h=b1.h, log_transform=True, warm_start=(f0.mu_rew, np.zeros((p, p))))
    assert e.value.code == "BOTH_STARTS_FAILED"


def test_table2_kl_pins_the_median_consistency_rule():
    """Table 2 (tests/golden/table2_kl_a09.json): A09, gamma = 50, n = 65536,
    alpha = 0.5, shift contamination, p = 4.  The KL deviation of the raw scatter the paper reports is
    reproduced when the h-subset covariance is rescaled so that the median squared robust distance of
    all n rows is chi2_{p,0.5} (the DetMCD implementations' rule), not with the c(alpha) factor of the
    text (our reading R1), which the oracle follows: under contamination the two
    differ (the h-subset is a central (h/n)/(1-eps) part of the inliers).  Finding F1 in DESIGN.md."""
    import json
    import os
    from oracle.chi2 import chi2_quantile
    from oracle.numerics import mahalanobis_sq
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table2_kl_a09.json")))

    def kl(A, B):
        M = A @ np.linalg.inv(B)
        return float(np.trace(M) - A.shape[0] - np.linalg.slogdet(M)[1])

    for eps in (0.1, 0.3):
        r1, med = [], []
        for rep in range(3):
            d = datagen.paper_simulation(4, eps, "shift", rep)
            n = d.X.shape[0]
            o = F.fit(d.X, alpha=0.5)
            S_h = o.Sigma_raw / consistency_factor((n // 2) / n, 4)
            d2 = mahalanobis_sq(d.X, o.mu_raw, S_h)
            r1.append(kl(o.Sigma_raw, d.sigma))
            med.append(kl(S_h * np.median(d2) / chi2_quantile(0.5, 4), d.sigma))
        paper = gold["IDC"][str(eps)]["shift"][0]
        assert abs(np.mean(med) / paper - 1.0) < 0.2, (eps, np.mean(med), paper)
        assert np.mean(r1) / paper < 0.8, (eps, np.mean(r1), paper)


def test_median_consistency_rule_invariant():
    """consistency="median": the raw scatter is rescaled so that the median squared robust distance of
    the block's rows under (mu_raw, Sigma_raw) is exactly chi2_{p,0.5} (F1); the h-subsets
    and the raw centre are those of the default rule."""
    from oracle.chi2 import chi2_quantile
    from oracle.numerics import mahalanobis_sq
    d = datagen.make_config(2, n=20_000)
    a = F.fit(d.X, h=d.h)
    m = F.fit(d.X, h=d.h, consistency="median")
    Z = (d.X - m.loc) / m.scale
    med = np.median(mahalanobis_sq(Z, m.mu_raw_z, m.Sigma_raw_z))
    assert med == pytest.approx(chi2_quantile(0.5, d.X.shape[1]), rel=1e-12)
    assert np.array_equal(a.blocks[0].starts[a.blocks[0].chosen].H, m.blocks[0].starts[m.blocks[0].chosen].H)
    assert np.allclose(a.mu_raw, m.mu_raw, rtol=0, atol=0)
    r = m.Sigma_raw / a.Sigma_raw
    assert np.allclose(r, r[0, 0], rtol=1e-12)  # a scalar multiple
    with pytest.raises(F.FitError):
        F.fit(d.X, h=d.h, consistency="other")


def test_reweighted_consistency_factor_p2():
    # Reading R17: Sigma_rew = c(0.975, p) * classical covariance of the
    # weighted rows.  On clean N(0, Sigma) data the reweighted RD^2 is then ~ chi2_p, so the flag rate
    # is 1 - 0.975 = 0.025 (binomial sd 0.00035 at n = 200k); without the factor it would be
    # P(chi2_2 > chi2_{2,.975} / c) = exp(-7.3778 / 2 / 1.1045) = 0.0354 at p = 2.  Also Sigma_rew
    # itself must estimate the generating Sigma (it is 1/1.1045 of it without the factor).
    S = np.array([[2.0, 0.6], [0.6, 0.5]])
    X = datagen.gaussian(200_000, 2, seed=41, sigma=S)
    r = F.fit(X, alpha=0.75)
    assert abs(r.flags.mean() - 0.025) < 0.0025
    ratio = np.trace(np.linalg.solve(S, r.Sigma_rew)) / 2
    assert abs(ratio - 1.0) < 0.02
