"""The bucketed univariate MCD (reading R4 for the reweighting) under its process-wide
switches, each read once per process, so every variant runs in a subprocess:
  * default: the reweighting sums fused into the gather pass (k_pr_final_fused decides the band values),
    CTAs per column from the column length;
  * RTD_UNI_NOFUSEDKEEP=1: the separate k_pr_keep pass;
  * RTD_PR_CTAS=4 / 32: other fixed CTA counts per column (another fold order of the partial sums);
  * short columns (4097..32768 rows): the fused cluster estimator (default) and RTD_UNI_CLUSTER_SPLIT=1 (the
    cluster sort followed by the one-CTA k_uni_small).
Every variant must give the oracle's window start exactly and its estimates to the parity tolerances."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N = 1_000_000


def _columns():
    rng = np.random.default_rng(31)
    return np.stack([rng.standard_normal(N), 100.0 + 3.0 * rng.standard_normal(N), np.exp(rng.standard_normal(N)),
                     np.concatenate([rng.standard_normal(N - N // 10), 9.0 + rng.standard_normal(N // 10)])])


SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np, torch
from paper_1910_05615_b200 import api
from tests.test_gpu_uni_variants import _columns
cols = _columns()
k0, s0 = api.counters()
g = api.unimcd(torch.from_numpy(cols).cuda())
k1, s1 = api.counters()
print("RESULT " + json.dumps({k: [float(v) for v in g[k]] for k in ("loc", "scale", "raw_loc", "raw_var")} |
                             {"start": [int(v) for v in g["start"]], "sorts": s1 - s0}))
""" % ROOT


@pytest.fixture(scope="module")
def oracle_fits():
    from oracle.unimcd import unimcd_reweighted
    return [unimcd_reweighted(c) for c in _columns()]


@pytest.mark.parametrize("env", [{}, {"RTD_UNI_NOFUSEDKEEP": "1"}, {"RTD_PR_CTAS": "4"},
                                 {"RTD_PR_CTAS": "32", "RTD_UNI_NOFUSEDKEEP": "1"}])
def test_unimcd_variants_match_oracle(env, oracle_fits):
    e = {k: v for k, v in os.environ.items() if not k.startswith("RTD_")}
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=e, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    g = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1][7:])
    assert g["sorts"] == 0
    for j, o in enumerate(oracle_fits):
        assert g["start"][j] == o.raw.start, j
        assert g["raw_loc"][j] == pytest.approx(o.raw.loc, rel=1e-15, abs=1e-300), j
        assert g["raw_var"][j] == pytest.approx(o.raw.var_raw, rel=1e-13), j
        assert g["loc"][j] == pytest.approx(o.loc, rel=1e-14, abs=1e-14), j
        assert g["scale"][j] == pytest.approx(o.scale, rel=1e-13), j


SHORT = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np, torch
from paper_1910_05615_b200 import api
rng = np.random.default_rng(5)
cols = np.stack([rng.standard_normal(20_000) * (1 + j) + j for j in range(16)])
g = api.unimcd(torch.from_numpy(cols).cuda())
print("RESULT " + json.dumps({k: [float(v) for v in g[k]] for k in ("loc", "scale", "raw_loc")} |
                             {"start": [int(v) for v in g["start"]]}))
""" % ROOT


@pytest.mark.parametrize("env", [{}, {"RTD_UNI_CLUSTER_SPLIT": "1"}])
def test_unimcd_short_column_variants_match_oracle(env):
    from oracle.unimcd import unimcd_reweighted
    e = {k: v for k, v in os.environ.items() if not k.startswith("RTD_")}
    e.update(env)
    r = subprocess.run([sys.executable, "-c", SHORT], env=e, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    g = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1][7:])
    rng = np.random.default_rng(5)
    cols = np.stack([rng.standard_normal(20_000) * (1 + j) + j for j in range(16)])
    for j in range(cols.shape[0]):
        o = unimcd_reweighted(cols[j])
        assert g["start"][j] == o.raw.start, j
        assert g["raw_loc"][j] == pytest.approx(o.raw.loc, rel=1e-15, abs=1e-300), j
        assert g["loc"][j] == pytest.approx(o.loc, rel=1e-14, abs=1e-14), j
        assert g["scale"][j] == pytest.approx(o.scale, rel=1e-13), j
