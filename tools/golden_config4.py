#!/usr/bin/env python
"""Writes tests/golden/config4_oracle.npz: the ORACLE's whole config-4 fit (BASELINE.json configs[3]).

Imports only `oracle/` and the seeded generator `paper_1910_05615_b200.datagen` (which holds none of
the method's arithmetic); nothing here touches the CUDA path.  The GPU test
tests/test_gpu_fullsize.py::test_config4_matches_oracle_golden compares the CUDA fit element by
element with this file.

Workload: n = 8,000,000, p = 40, h = 6,000,000, q = 8 contiguous per-shard blocks (the bench.py
workload; BASELINE.json: "rows sharded evenly ... with per-shard DetMCD"), seed 191005615.
The fit follows PAPER.md:746-1043 (§4 steps 1-10) step by step (oracle/fit.py).

Stored (X units unless stated; flags/subsets as packed bit masks over the n rows):
  loc, scale                      univariate reweighted MCD per column
  mu_raw, sigma_raw               pooled raw fit
  mu_rew, sigma_rew, n_weighted   reweighted fit
  cutoff2                         chi2_{p,0.975}
  block_chosen, block_logdet      per block: chosen start (0 wrapping / 1 GSSCM), its log det (z units)
  start_steps, start_logdet       per (block, start)
  hsubset_bits                    1 iff the row is in its block's chosen h-subset
  hsub_band_rows                  rows whose oracle distance lies within 1e-9 (relative) of their
                                  block's h-th distance (exempt from subset comparison, reading Q23)
  weights_bits, flags_bits        reweighting weights / flags
  flag_band_rows                  rows whose final RD lies within 1e-9 (relative) of c_p
  weight_band_rows                rows whose raw RD lies within 1e-9 (relative) of c_p
  rd2_idx, rd2_val                final RD^2 of every 997th row
  x_digest                        sha256 of X's bytes (the generator must reproduce them exactly)

Usage: python tools/golden_config4.py [--out tests/golden/config4_oracle.npz]   (~10-20 min of CPU)
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import fit as ofit  # noqa: E402
from oracle.numerics import mahalanobis_sq  # noqa: E402
from paper_1910_05615_b200 import datagen  # noqa: E402

SEED = 191005615
BAND = 1e-9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "config4_oracle.npz"))
    a = ap.parse_args()
    t0 = time.time()
    d = datagen.make_config(4)
    X = d.X
    n, p = X.shape
    print(f"generated {n} x {p} in {time.time() - t0:.0f} s", flush=True)
    o = ofit.fit(X, h=d.h, q=d.q, seed=SEED, log_transform=d.log_transform, partition_mode="contiguous")
    print(f"oracle fit done at {time.time() - t0:.0f} s", flush=True)
    q = d.q
    hs = np.zeros(n, dtype=bool)
    band_rows = []
    chosen, blogdet, steps, slogdet = [], [], [], []
    Z = (X - o.loc) / o.scale
    for b in o.blocks:
        chosen.append(b.chosen)
        blogdet.append(b.logdet)
        steps.append([s.steps for s in b.starts])
        slogdet.append([s.logdet for s in b.starts])
        st = b.starts[b.chosen]
        hs[b.rows[st.H]] = True
        dd = np.sqrt(np.maximum(mahalanobis_sq(Z[b.rows], st.mu, st.Sigma), 0.0))
        dh = np.sort(dd)[b.h - 1]
        band_rows.append(b.rows[np.abs(dd - dh) <= BAND * dh])
    del Z
    cp = np.sqrt(o.cutoff2)
    drd = np.sqrt(np.maximum(o.rd2, 0.0))
    flag_band = np.nonzero(np.abs(drd - cp) <= BAND * cp)[0]
    d2raw = mahalanobis_sq(X, o.mu_raw, o.Sigma_raw)
    draw = np.sqrt(np.maximum(d2raw, 0.0))
    weight_band = np.nonzero(np.abs(draw - cp) <= BAND * cp)[0]
    idx = np.arange(0, n, 997)
    np.savez_compressed(
        a.out,
        loc=o.loc, scale=o.scale, mu_raw=o.mu_raw, sigma_raw=o.Sigma_raw, mu_rew=o.mu_rew, sigma_rew=o.Sigma_rew,
        n_weighted=np.int64(o.weights.sum()), cutoff2=np.float64(o.cutoff2), kept_blocks=np.array(o.kept_blocks),
        block_chosen=np.array(chosen), block_logdet=np.array(blogdet), start_steps=np.array(steps),
        start_logdet=np.array(slogdet), hsubset_bits=np.packbits(hs),
        hsub_band_rows=np.concatenate(band_rows).astype(np.int64),
        weights_bits=np.packbits(o.weights), flags_bits=np.packbits(o.flags),
        flag_band_rows=flag_band.astype(np.int64), weight_band_rows=weight_band.astype(np.int64),
        rd2_idx=idx.astype(np.int64), rd2_val=o.rd2[idx],
        n=np.int64(n), p=np.int64(p), h=np.int64(d.h), q=np.int64(q),
        x_digest=np.frombuffer(hashlib.sha256(X.tobytes()).digest(), dtype=np.uint8))
    print(f"wrote {a.out} at {time.time() - t0:.0f} s: chosen {chosen}, steps {steps}, "
          f"band rows {sum(len(r) for r in band_rows)} / flag band {len(flag_band)}", flush=True)


if __name__ == "__main__":
    main()
