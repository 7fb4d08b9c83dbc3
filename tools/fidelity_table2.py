"""Paper-fidelity harness: Table 2 of the paper (A09 Sigma, gamma = 50,
n = 65536, alpha = 0.5; point / shift / cluster contamination at eps = 0.1, 0.3; p = 4, 8, 16),
KL deviation KL(A, B) = tr(A B^-1) - p - log det(A B^-1) of the estimated scatter from the true one
(PAPER.md:1150-1160), averaged over replications, for IDC (q = 1) and IDCP_4 (q = 4) run on the
CUDA path through the public API.

Reported per cell: KL of the raw scatter (c(alpha)-scaled, reading R1 -- the text's definition,
PAPER.md:158-175), KL of the reweighted scatter, and KL of the raw scatter of the fit with
consistency = RTD_CONS_MEDIAN (the h-subset covariance rescaled so that the median squared robust
distance of the block's rows equals chi2_{p,0.5}, the rule of the DetMCD implementations; F1).  The paper's
IDC / IDCP_4 values (tests/golden/table2_kl_a09.json) are printed beside them.

  python tools/fidelity_table2.py [--reps 50] [--out profiles/r01_fidelity_table2.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def kl(A, B):
    M = A @ np.linalg.inv(B)
    s, ld = np.linalg.slogdet(M)
    return float(np.trace(M) - A.shape[0] - ld)


def main():
    import torch

    from paper_1910_05615_b200 import api, datagen
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01_fidelity_table2.json"))
    a = ap.parse_args()
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "table2_kl_a09.json")))
    rows = []
    t0 = time.time()
    for eps in (0.1, 0.3):
        for kind in ("point", "shift", "cluster"):
            for pi, p in enumerate((4, 8, 16)):
                acc = {"IDC": {"raw": [], "rew": [], "med": []}, "IDCP4": {"raw": [], "rew": [], "med": []}}
                for rep in range(a.reps):
                    d = datagen.paper_simulation(p, eps, kind, rep)
                    n = d.X.shape[0]
                    Xd = torch.from_numpy(d.X).to("cuda:0")
                    for var, q in (("IDC", 1), ("IDCP4", 4)):
                        g = api.fit(Xd, alpha=0.5, q=q, seed=1000 + rep, outputs=())
                        acc[var]["raw"].append(kl(g.sigma_raw, d.sigma))
                        acc[var]["rew"].append(kl(g.sigma_rew, d.sigma))
                        gm = api.fit(Xd, alpha=0.5, q=q, seed=1000 + rep, outputs=(), consistency=1)
                        acc[var]["med"].append(kl(gm.sigma_raw, d.sigma))
                for var in ("IDC", "IDCP4"):
                    paper = gold[var][str(eps)][kind][pi]
                    r = {k: float(np.mean(v)) for k, v in acc[var].items()}
                    rows.append({"variant": var, "eps": eps, "kind": kind, "p": p, "reps": a.reps,
                                 "kl_raw_R1": r["raw"], "kl_rew": r["rew"], "kl_raw_median_rule": r["med"],
                                 "paper": paper, "ratio_R1": r["raw"] / paper, "ratio_median_rule": r["med"] / paper})
                    print(f"{var:6s} eps={eps} {kind:8s} p={p:2d}  R1 {r['raw']:.5f}  rew {r['rew']:.5f}  "
                          f"median-rule {r['med']:.5f}  paper {paper:.5f}", flush=True)
    out = {"table": "PAPER.md Table 2 (tbl:KL_A09), panel A", "design": "PAPER.md:1102-1184",
           "generator": "datagen.paper_simulation", "path": "api.fit on cuda:0 (the CUDA path)",
           "wall_s": time.time() - t0, "rows": rows}
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
