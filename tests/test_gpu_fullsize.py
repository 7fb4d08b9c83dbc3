"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration bench.py times.

* Config 3 (n = 1,000,000, p = 20, h = 500,001, q = 1): the whole oracle fit
  (about 80 s of CPU) against the CUDA fit, element by element (T3).
* Config 4 (n = 8,000,000, p = 40, q = 8 contiguous per-shard blocks, the
  bench workload): the oracle cannot re-run the whole fit in seconds, so the
  test checks what holds at any size, computed by the oracle's own routines
  from the GPU's per-row outputs:
    - sampled columns' univariate reweighted MCD (loc, scale) recomputed by the
      oracle;
    - each block's returned h-subset is a C-step fixed point: the h_l smallest
      distances under the mean / covariance of that very subset are the subset
      itself (convergence H_new == H_old, reading R12);
    - the raw fit equals the oracle's median / KL / pooling
      of the per-block c(alpha_l)-scaled subset moments;
    - the reweighted fit and the weights equal the oracle's reweighting under
      that raw fit, and the flags and RD^2 of all
      n rows equal the oracle's flag pass.
  Everything is compared in original X units: the subset moments, the pooling
  and the Mahalanobis distances are affine equivariant (reading R22), so no
  GPU-computed standardisation enters the oracle side.
* The whole oracle fit of config 4, precomputed by tools/golden_config4.py (oracle/ + the seeded
  generator only) into tests/golden/config4_oracle.npz, compared element by element.
* An opt-in (RTD_FULLSIZE_SLOW=1) case reruns the oracle's whole block fit of
  block 0 of config 4 (global standardisation over 8M rows, both starts,
  C-steps: several minutes of CPU) and compares its h-subset with the GPU's.
"""
import math
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fit as ofit  # noqa: E402
from oracle.chi2 import chi2_quantile, consistency_factor  # noqa: E402
from oracle.cstep import h_subset, mean_cov  # noqa: E402
from oracle.numerics import mahalanobis_sq  # noqa: E402
from oracle.parallel import partition, select_and_pool  # noqa: E402
from oracle.unimcd import unimcd_reweighted  # noqa: E402
from paper_1910_05615_b200 import api, datagen  # noqa: E402
from tests._parity import TOL, assert_flags_equal, assert_subset_equal, rel_mu, rel_sigma  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
SEED = 191005615


@pytest.fixture(scope="module")
def cfg4():
    d = datagen.make_config(4)
    Xd = torch.from_numpy(d.X).to(DEV)
    # bench.py's call: contiguous per-shard blocks, q = 8, all rows on one GPU
    g = api.fit(Xd, h=d.h, q=d.q, seed=SEED, log_transform=d.log_transform, partition=1)
    torch.cuda.synchronize()
    del Xd
    return d, g


def test_config3_full_size_matches_oracle():
    from tests.test_gpu_parity import _compare_fit
    d = datagen.make_config(3)
    assert d.X.shape == (1_000_000, 20)
    g = api.fit(torch.from_numpy(d.X).to(DEV), h=d.h)
    o = ofit.fit(d.X, h=d.h)
    _compare_fit(g, o, d.X)
    assert g.warnings & 1  # RTD_W_H_BELOW_BOUND: h = 500,001 < [(n+p+1)/2] (reading R24)
    assert [int(s) for s in g.start_steps] == [b.steps for b in o.blocks[0].starts]


def test_config4_sampled_columns_standardisation(cfg4):
    d, g = cfg4
    for j in (0, 17, 39):
        u = unimcd_reweighted(d.X[:, j])
        assert g.loc[j] == pytest.approx(u.loc, rel=1e-13, abs=1e-14)
        assert g.scale[j] == pytest.approx(u.scale, rel=1e-12)


def test_config4_blocks_fixed_point_pool_reweight_flags(cfg4):
    d, g = cfg4
    X = d.X
    n, p = X.shape
    q = d.q
    block, pos, m = partition(n, q, SEED, "contiguous")
    hb = (d.h * m) // n
    assert (g.q, g.m, g.h_block) == (q, m, hb)
    hs = g.hsubset.cpu().numpy().astype(bool)
    calpha = consistency_factor(hb / m, p)
    mus, Ss = [], []
    for b in range(q):
        rows = np.arange(b * m, (b + 1) * m)
        assert np.all(block[rows] == b)
        Xb = X[rows]
        Hb = np.nonzero(hs[rows])[0]
        assert Hb.size == hb
        mu_b, S_b = mean_cov(Xb, Hb)
        d2 = mahalanobis_sq(Xb, mu_b, S_b)
        # C-step fixed point: H_new == H_old (tie band of the north star)
        assert_subset_equal(hs[rows], h_subset(d2, hb), d2, hb)
        mus.append(mu_b)
        Ss.append(calpha * S_b)
    assert not hs[q * m:].any()
    assert g.n_valid_blocks == q
    mu_raw, S_raw, kept, _ = select_and_pool(mus, Ss, [m] * q, list(range(q)))
    assert g.n_kept_blocks == len(kept) == math.ceil(q / 2)
    assert rel_sigma(g.sigma_raw, S_raw) < TOL
    assert rel_mu(g.mu_raw, mu_raw, S_raw) < TOL
    # reweighting over the fitted rows under the raw fit
    c2 = chi2_quantile(0.975, p)
    fitted = block >= 0
    d2raw = mahalanobis_sq(X, mu_raw, S_raw)
    w = fitted & (d2raw <= c2)
    assert_flags_equal(g.weights.cpu().numpy(), w, d2raw, c2)
    Xw = X[w]
    mu_rew = Xw.mean(axis=0)
    D = Xw - mu_rew
    S_rew = consistency_factor(0.975, p) * (D.T @ D) / (w.sum() - 1)
    del Xw, D
    assert g.n_weighted == int(w.sum())
    assert rel_sigma(g.sigma_rew, S_rew) < TOL
    assert rel_mu(g.mu_rew, mu_rew, S_rew) < TOL
    # flag pass over all n rows
    rd2 = mahalanobis_sq(X, mu_rew, S_rew)
    assert_flags_equal(g.flags.cpu().numpy(), rd2 > c2, rd2, c2)
    assert np.allclose(g.rd2.cpu().numpy(), rd2, rtol=1e-9, atol=1e-9)
    # the shift rows (Mahalanobis 8 vs cut-off 7.7) are flagged; the tight cluster N(m, 0.05^2 Sigma) at
    # Mahalanobis 8 lies inside the DetMCD h-subsets at p = 40, h = 0.75 n -- the oracle does the same
    # (tests/test_oracle_fit.py::test_config4_recipe_cluster_absorbed), a property of the estimator
    fl = g.flags.cpu().numpy().astype(bool)
    assert fl[d.meta["shift_rows"]].mean() > 0.99
    assert fl[~d.outliers].mean() < 0.06


def test_config4_matches_oracle_golden(cfg4):
    """The WHOLE oracle fit of config 4 (tests/golden/config4_oracle.npz, written by
    tools/golden_config4.py, which imports only oracle/ and the seeded generator; ~20 min of CPU)
    against the CUDA fit of the bench workload, element by element: global standardisation
    (PAPER.md:430-453, 756-766), every (block, start)'s converged log det and C-step count, the chosen
    start and its h-subset per block, the pooled raw fit, the
    reweighted fit and weights, the flags and sampled RD^2 of all n rows
    (PAPER.md:217-220).  Tie bands of reading Q23 come from the oracle's own distances."""
    import hashlib
    d, g = cfg4
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "config4_oracle.npz"))
    n, p, q = int(z["n"]), int(z["p"]), int(z["q"])
    assert d.X.shape == (n, p) and d.h == int(z["h"]) and d.q == q
    assert hashlib.sha256(d.X.tobytes()).digest() == z["x_digest"].tobytes(), "generator drift: regenerate the golden"
    assert np.allclose(g.loc, z["loc"], rtol=1e-13, atol=1e-14)
    assert np.allclose(g.scale, z["scale"], rtol=1e-12, atol=0)
    # per (block, start): converged log det (update-based on the GPU, reading R12) and C-step count
    sl = np.asarray(g.start_logdet).reshape(q, 2)
    assert np.allclose(sl, z["start_logdet"], rtol=1e-12, atol=0)
    assert np.array_equal(np.asarray(g.start_steps).reshape(q, 2), z["start_steps"])
    assert [int(c) for c in g.block_chosen] == [int(c) for c in z["block_chosen"]]
    # chosen h-subsets of all blocks, in original row order (exempt: rows in the oracle's tie band)
    hs_o = np.unpackbits(z["hsubset_bits"])[:n].astype(bool)
    hs_g = g.hsubset.cpu().numpy().astype(bool)
    diff = np.nonzero(hs_o != hs_g)[0]
    assert np.isin(diff, z["hsub_band_rows"]).all(), f"{diff.size} subset rows differ outside the tie band"
    assert hs_g.sum() == hs_o.sum()
    # pooled raw and reweighted fits (X units, north-star tolerance)
    assert rel_sigma(g.sigma_raw, z["sigma_raw"]) < TOL
    assert rel_mu(g.mu_raw, z["mu_raw"], z["sigma_raw"]) < TOL
    assert rel_sigma(g.sigma_rew, z["sigma_rew"]) < TOL
    assert rel_mu(g.mu_rew, z["mu_rew"], z["sigma_rew"]) < TOL
    assert g.n_kept_blocks == len(z["kept_blocks"])
    w_o = np.unpackbits(z["weights_bits"])[:n].astype(bool)
    wd = np.nonzero(w_o != g.weights.cpu().numpy().astype(bool))[0]
    assert np.isin(wd, z["weight_band_rows"]).all(), f"{wd.size} weights differ outside the tie band"
    assert abs(g.n_weighted - int(z["n_weighted"])) <= len(z["weight_band_rows"])
    f_o = np.unpackbits(z["flags_bits"])[:n].astype(bool)
    fd = np.nonzero(f_o != g.flags.cpu().numpy().astype(bool))[0]
    assert np.isin(fd, z["flag_band_rows"]).all(), f"{fd.size} flags differ outside the tie band"
    idx = z["rd2_idx"]
    assert np.allclose(g.rd2.cpu().numpy()[idx], z["rd2_val"], rtol=1e-9, atol=1e-9)


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("RTD_FULLSIZE_SLOW") != "1", reason="opt-in: several minutes of oracle CPU")
def test_config4_block0_full_oracle(cfg4):
    d, g = cfg4
    X = d.X
    n, p = X.shape
    loc, scale = ofit.standardize(X)
    assert np.allclose(g.loc, loc, rtol=1e-13, atol=1e-14) and np.allclose(g.scale, scale, rtol=1e-12)
    m = n // d.q
    hb = (d.h * m) // n
    Zb = (X[:m] - loc) / scale
    starts, chosen = ofit.fit_block(Zb, hb)
    assert chosen >= 0 and int(g.block_chosen[0]) in (0, 1)
    st = starts[chosen]
    d2 = mahalanobis_sq(Zb, st.mu, st.Sigma)
    assert_subset_equal(g.hsubset.cpu().numpy()[:m], st.H, d2, hb)
    assert [int(s) for s in g.start_steps[:2]] == [s.steps for s in starts]
