"""Table 1 ablation ladder on the B200.

The paper switches its modifications on one after the other: new Initial estimators (I), Distances by
the Cholesky factor (D), update-based C-steps (C), Parallelisation into q blocks (P).  DetMCD itself
(six starts) is out of scope; the ladder here is, through the public API on cuda:0:

  I       distance=RTD_DIST_INVERSE, refresh_every=1 (explicit inverse, plain recompute every C-step)
  ID      distance=RTD_DIST_CHOLESKY, refresh_every=1
  IDC     the default serial fit (Cholesky distances, update-based C-steps)
  IDC+SMW distance=RTD_DIST_SMW: the inverse and log det updated by Sherman-Morrison-Woodbury on the
          C-steps that interchange exactly two cases, distances by the inverse
  IDCP_q  IDC on q blocks (contiguous blocks, the bench partition)

for a BASELINE config, timed with CUDA events per fit (warm-up first), with the per-kernel-class device
time of one profiled fit.

  python tools/ablation.py [--config 4] [--reps 3] [--q 8] [--out profiles/r01_ablation_cfg4.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    from paper_1910_05615_b200 import api, datagen
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--q", type=int, default=8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    d = datagen.make_config(a.config)
    n, p = d.X.shape
    Xd = torch.from_numpy(d.X).to("cuda:0")
    variants = [("I", dict(distance=1, refresh_every=1, q=1)), ("ID", dict(distance=0, refresh_every=1, q=1)),
                ("IDC", dict(q=1)), ("IDC+SMW", dict(distance=2, q=1)), (f"IDCP_{a.q}", dict(q=a.q, partition=1))]
    out = {"config": a.config, "n": n, "p": p, "h": d.h, "reps": a.reps, "table": "PAPER.md:1076-1100 (Table 1)",
           "variants": {}}
    stream = torch.cuda.current_stream()
    for name, kw in variants:
        def one():
            return api.fit(Xd, h=d.h, seed=191005615, log_transform=d.log_transform, outputs=("flags",), **kw)
        one()
        torch.cuda.synchronize()
        ms = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g = one()
            e1.record(stream)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
        api.set_profiling(True)
        one()
        prof = api.profile()
        api.set_profiling(False)
        t = float(np.median(ms))
        out["variants"][name] = {"opts": kw, "ms_per_fit": t, "obs_per_s": n / (t / 1e3),
                                 "start_steps": [int(x) for x in g.start_steps],
                                 "breakdown_ms": {k: v["ms"] for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}
        print(f"{name:8s} {t:9.2f} ms/fit  {n / (t / 1e3) / 1e6:8.2f} M obs/s  steps {list(g.start_steps)}", flush=True)
    base = out["variants"]["I"]["ms_per_fit"]
    for name in out["variants"]:
        out["variants"][name]["speedup_vs_I"] = base / out["variants"][name]["ms_per_fit"]
    path = a.out or os.path.join(ROOT, "profiles", f"r01_ablation_cfg{a.config}.json")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
