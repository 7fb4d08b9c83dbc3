"""Pins for oracle/unimcd.py: brute force over all h-subsets, exact windows, SPEC examples."""
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle.chi2 import consistency_factor
from oracle.unimcd import DegenerateScale, unimcd_raw, unimcd_reweighted

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))


def _brute_all_subsets(x, h):
    """Exact raw MCD over ALL C(n,h) subsets (not only contiguous windows)."""
    best = None
    for S in itertools.combinations(range(len(x)), h):
        v = [Fraction(float(x[i])) for i in S]
        m = sum(v) / h
        ss = sum((a - m) ** 2 for a in v)
        if best is None or ss < best[0]:
            best = (ss, m)
    return best


@pytest.mark.parametrize("seed", range(6))
def test_raw_matches_all_subsets_bruteforce(seed):
    # the univariate optimum is a contiguous window of the sorted data
    rng = np.random.default_rng(seed)
    n = 9 + seed % 3
    x = rng.standard_normal(n) * (1 + seed)
    if seed % 2:
        x[:2] += 25.0
    h = n // 2 + 1
    ss, m = _brute_all_subsets(x, h)
    r = unimcd_raw(x, h)
    assert r.loc == pytest.approx(float(m), rel=1e-15, abs=1e-15)
    assert r.var_raw == pytest.approx(float(ss / (h - 1)), rel=1e-15)


def test_spec_raw_example():
    g = GOLD["spec_examples"]["unimcd_raw"]
    r = unimcd_raw(np.array(g["x"], float), g["h"])
    assert r.start == 0          # tie (0,1,2) vs (1,2,3) -> lowest start
    assert r.loc == g["loc"]
    assert math.sqrt(r.var_raw) == g["sd_raw"]


def test_spec_reweighted_example():
    g = GOLD["spec_examples"]["unimcd_rew"]
    u = unimcd_reweighted(np.array(g["x"], float))
    assert u.loc == g["loc"]
    assert u.n_kept == 5
    # kept {0,...,4}: var = 2.5, times c(0.975, 1)
    assert u.scale == pytest.approx(math.sqrt(2.5 * consistency_factor(0.975, 1)), rel=1e-15)


def test_degenerate():
    with pytest.raises(DegenerateScale):
        unimcd_reweighted(np.full(10, 3.0))
    with pytest.raises(DegenerateScale):
        unimcd_reweighted(np.array([1.0, 1, 1, 1, 1e6]))


def _exact_argmin_all_windows(x, h):
    y = sorted(Fraction(float(v)) for v in x)
    best = None
    for s in range(len(y) - h + 1):
        w = y[s:s + h]
        m = sum(w) / h
        v = sum((a - m) ** 2 for a in w)
        if best is None or v < best[0]:
            best = (v, s)
    return best[1]


@pytest.mark.parametrize("seed", range(4))
def test_window_argmin_is_exact(seed):
    rng = np.random.default_rng(100 + seed)
    x = rng.standard_normal(301) + 1e3 * (seed == 3)   # large offset stresses cancellation
    assert unimcd_raw(x, 151).start == _exact_argmin_all_windows(x, 151)


def test_symmetric_exact_tie_takes_lowest_start():
    # mirror-symmetric sample: windows s and n-h-s have exactly equal SQ
    rng = np.random.default_rng(7)
    a = np.sort(np.abs(rng.standard_normal(200))) + 0.01
    x = np.concatenate([-a, a])
    h = x.size // 2 + 1
    r = unimcd_raw(x, h)
    s_exact = _exact_argmin_all_windows(x, h)
    assert r.start == s_exact
    assert r.start <= x.size - h - r.start       # the lower of the mirrored pair


def test_power_of_two_equivariance_exact():
    rng = np.random.default_rng(11)
    x = rng.standard_normal(5001)
    u = unimcd_reweighted(x)
    for k in (-3, 1, 7):
        v = unimcd_reweighted(x * 2.0 ** k)
        assert v.loc == u.loc * 2.0 ** k
        assert v.scale == u.scale * 2.0 ** k
    w = unimcd_reweighted(-x)
    assert w.loc == -u.loc and w.scale == u.scale


def test_translation_equivariance():
    rng = np.random.default_rng(12)
    x = rng.standard_normal(4001)
    u = unimcd_reweighted(x)
    v = unimcd_reweighted(x + 17.25)
    assert v.loc == pytest.approx(u.loc + 17.25, abs=1e-12)
    assert v.scale == pytest.approx(u.scale, rel=1e-10)


def test_gaussian_consistency():
    # N(0,1), n = 1e5 -> loc 0 +- 0.02, scale 1 +- 0.03
    rng = np.random.default_rng(13)
    u = unimcd_reweighted(rng.standard_normal(100_000))
    assert abs(u.loc) < 0.02 and abs(u.scale - 1) < 0.03


def test_breakdown():
    rng = np.random.default_rng(14)
    x = rng.standard_normal(1001)
    base = unimcd_reweighted(x)
    y = x.copy()
    y[: 1001 - (1001 // 2 + 1)] = 1e9
    bad = unimcd_reweighted(y)
    assert abs(bad.loc - base.loc) < 5 * base.scale
