#!/usr/bin/env python
"""Modelled multi-GPU scaling of the sharded config-4 fit, from per-rank stage timings on ONE B200.

This run has one GPU, so `bench.py --gpus N` (rtdetmcd_fit_sharded over NCCL) cannot be timed here.  This
tool times, on one GPU and through the library's stage entry points, exactly the work rank 0 of G ranks does
in rtdetmcd_fit_sharded:
  * the univariate MCD of its ceil(p/G) owned columns over all n rows (global standardisation),
  * rtdetmcd_blocks_fit on its n/G rows = q/G blocks (H0 transpose, Z, starts, refinement, C-steps),
  * rtdetmcd_blocks_reweight on those blocks and rtdetmcd_flag on its n/G rows,
and adds a MODEL of the exchanges: the column all-to-all (C2) moves (G-1)/G of the rank's n/G x p x 8 bytes
each way at `--link-gbs` (NVLink 5: 900 GB/s per direction per GPU, derated by --link-eff), plus a fixed
latency per collective for C3-C5 and the agreement words.  The result is a model (stated as such in the JSON),
not a measurement: T_G = max-rank compute (rank 0 holds the most columns) + modelled communication, and
speedup = T_1 / T_G with T_1 = the measured single-GPU rtdetmcd_fit of the same q blocks (q = 8, the bench's
block count; q = 48, the paper's partition rule for config 4).

Usage: python tools/scaling_model.py [--out profiles/r02_scaling_model.json]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_1910_05615_b200 import api, datagen
    from paper_1910_05615_b200._lib import lib

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_scaling_model.json"))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--link-gbs", type=float, default=900.0)
    ap.add_argument("--link-eff", type=float, default=0.7)
    ap.add_argument("--coll-latency-us", type=float, default=30.0)
    ap.add_argument("--q", type=int, nargs="+", default=[8, 48],
                    help="block counts: 8 (SURVEY Q18, the bench) and 48 (the paper's rule, PAPER.md:1394-1403)")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    d = datagen.make_config(4)
    n, p = d.X.shape
    h = d.h
    X = torch.from_numpy(d.X).cuda()
    L = lib()
    ctx = api.new_context(0)
    stream = torch.cuda.current_stream()

    def timed(fn):
        ts = []
        for _ in range(a.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        return float(np.median(ts[1:]))

    fl = torch.empty(n, dtype=torch.uint8, device="cuda")
    Xc = X.t().contiguous()  # (p, n) column-major columns for the univariate MCD stage
    models = []
    for q in a.q:
        t1 = timed(lambda: api.fit(X, h=h, q=q, partition=1, outputs=(), out_buffers={"flags": fl}))
        g = api.fit(X, h=h, q=q, partition=1)
        loc, scale = np.ascontiguousarray(g.loc), np.ascontiguousarray(g.scale)
        rows = []
        for G in (1, 2, 4, 8):
            cpr = math.ceil(p / G)
            nl = n // G
            ql = q // G
            m = n // q
            hb = (h * m) // n
            cols = Xc[:cpr].contiguous()
            t_std = timed(lambda: api.unimcd(cols, ctx=ctx))
            Xl = X[:nl].contiguous()
            opts = api.default_opts(h=h)
            rec = np.zeros((ql, 4 + p + p * p))

            def blocks():
                rc = L.rtdetmcd_blocks_fit(ctx["h"], C.c_void_p(Xl.data_ptr()), nl, p, loc.ctypes.data,
                                           scale.ctypes.data, ql, q, hb, C.byref(opts), rec.ctypes.data)
                assert rc == 0, L.rtdetmcd_last_error(ctx["h"])
            t_blocks = timed(blocks)
            # reweighting needs the session's raw fit: aggregate rank 0's records repeated as the q-block set
            allrec = np.ascontiguousarray(np.concatenate([rec] * G))
            mu, sg, nk = np.zeros(p), np.zeros((p, p)), C.c_int32()
            sums = np.zeros((ql, L.rtdetmcd_moment_doubles(p)))

            def rew():
                blocks()
                assert L.rtdetmcd_aggregate(ctx["h"], q, p, m, allrec.ctypes.data, mu.ctypes.data, sg.ctypes.data,
                                            C.byref(nk)) == 0
                assert L.rtdetmcd_blocks_reweight(ctx["h"], 0.975, sums.ctypes.data, None) == 0
            t_rew = max(0.0, timed(rew) - t_blocks)
            t_flag = timed(lambda: api.flag(Xl, g.mu_rew, g.sigma_rew, want_rd2=False, ctx=ctx))
            bytes_c2 = (G - 1) / G * nl * p * 8 if G > 1 else 0.0
            t_c2 = bytes_c2 / (a.link_gbs * 1e9 * a.link_eff) * 1e3
            t_coll = (5 * a.coll_latency_us * 1e-3) if G > 1 else 0.0
            tg = t_std + t_blocks + t_rew + t_flag + t_c2 + t_coll
            rows.append({"gpus": G, "blocks_per_gpu": ql, "ms_std_owned_columns": t_std, "ms_blocks": t_blocks,
                         "ms_reweight": t_rew, "ms_flag": t_flag, "ms_c2_model": t_c2, "ms_collectives_model": t_coll,
                         "ms_total_model": tg, "obs_per_s_model": n / (tg / 1e3), "speedup_vs_1gpu_fit": t1 / tg})
            print(json.dumps({"q": q, **rows[-1]}), flush=True)
        models.append({"q": q, "ms_single_gpu_fit": t1, "rows": rows})
    out = {"kind": "MODEL (per-rank stage times measured on one B200 + modelled exchanges), not a multi-GPU run",
           "workload": "cfg4_n8M_p40 contiguous blocks, rank 0 of G (it owns the most columns)",
           "link_gbs": a.link_gbs, "link_eff": a.link_eff, "coll_latency_us": a.coll_latency_us, "models": models}
    json.dump(out, open(a.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
