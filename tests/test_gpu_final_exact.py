"""Reading R12's optional exact final recompute (RTD_FINAL_EXACT=1, read once per process, so it runs in a
subprocess): the winning start of every block gets its (mu, Sigma, log det) recomputed densely from its
final h-subset (eqs. of the plain C-step) instead of keeping the update-based sums
(PAPER.md:685-713).  Both must match the oracle's plain recompute to the north-star tolerance, and agree
with each other to ~1e-13."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import torch
from paper_1910_05615_b200 import api, datagen
out = {}
for cfg, n, q in ((2, 100_000, 1), (4, 40_000, 4)):
    d = datagen.make_config(cfg, n=n)
    h = d.h if cfg == 2 else int(0.75 * n)
    g = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1, outputs=("flags",))
    out[f"{cfg}"] = {"sigma_raw": g.sigma_raw.tolist(), "mu_raw": g.mu_raw.tolist(), "sigma_rew": g.sigma_rew.tolist(),
                     "mu_rew": g.mu_rew.tolist(), "start_logdet": [float(v) for v in g.start_logdet],
                     "flags": int(g.flags.sum().item())}
print("RESULT " + json.dumps(out))
""" % ROOT


def _run(final_exact: bool):
    env = dict(os.environ)
    env.pop("RTD_FINAL_EXACT", None)
    if final_exact:
        env["RTD_FINAL_EXACT"] = "1"
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_final_exact_recompute_matches_oracle_and_update_based():
    from oracle import fit as ofit
    from paper_1910_05615_b200 import datagen
    from tests._parity import TOL, rel_mu, rel_sigma
    ex, up = _run(True), _run(False)
    for cfg, n, q in ((2, 100_000, 1), (4, 40_000, 4)):
        d = datagen.make_config(cfg, n=n)
        h = d.h if cfg == 2 else int(0.75 * n)
        o = ofit.fit(d.X, h=h, q=q, partition_mode="contiguous")
        for res in (ex[str(cfg)], up[str(cfg)]):
            assert rel_sigma(np.array(res["sigma_raw"]), o.Sigma_raw) < TOL
            assert rel_mu(np.array(res["mu_raw"]), o.mu_raw, o.Sigma_raw) < TOL
            assert rel_sigma(np.array(res["sigma_rew"]), o.Sigma_rew) < TOL
            assert res["flags"] == int(o.flags.sum())
        a, b = np.array(ex[str(cfg)]["sigma_raw"]), np.array(up[str(cfg)]["sigma_raw"])
        assert rel_sigma(a, b) < 1e-12
        ld_o = [s.logdet for blk in o.blocks for s in blk.starts]
        assert np.allclose(ex[str(cfg)]["start_logdet"], ld_o, rtol=0, atol=1e-11)
