"""Launch-by-launch error check of the product path (SURVEY §4 T6's sanitizer run; compute-sanitizer is closed
on this GPU pool): small fits -- config 1 (one-CTA C-step loop), a config-5 batch (cluster kernels: the
univariate estimator and the C-step loop), a blocked config-4 sample (TMA distance / moment / GEMM kernels,
select with candidate mode, bucketed univariate MCD) and the flag pass -- each compared with the oracle.
Run as: RTD_DEBUG_SYNC=1 python tools/launch_check.py  (a device synchronisation and error check after every
launch: an out-of-bounds access or a trap surfaces at the kernel that caused it)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1910_05615_b200 import api, datagen  # noqa: E402
from oracle import fit as ofit  # noqa: E402

cases = [(1, None, 1), (5, 20_000, 1), (4, 140_000, 2)]
for cfg, n, q in cases:
    d = datagen.make_config(cfg, n=n) if n else datagen.make_config(cfg)
    h = d.h if cfg != 4 else int(0.75 * d.X.shape[0])
    g = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1, log_transform=d.log_transform)
    torch.cuda.synchronize()
    o = ofit.fit(d.X, h=h, q=q, partition_mode="contiguous", log_transform=d.log_transform)
    rel = np.linalg.norm(g.sigma_rew - o.Sigma_rew) / np.linalg.norm(o.Sigma_rew)
    print(f"config {cfg} n={d.X.shape[0]} q={q}: rel(Sigma_rew) = {rel:.2e}", flush=True)
    assert rel < 1e-10
print("sanitize run ok")
