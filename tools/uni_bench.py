#!/usr/bin/env python
"""Time the univariate-MCD stage (rtdetmcd_unimcd, the pruned exact window + reweighting) on the two column
shapes of a config-4 fit: the standardisation's 40 columns of 8M rows and a refinement call's 640 columns of
1M rows.  CUDA events around each call (which ends with a host read of the
results), median over --reps after one warm-up call.

Usage: python tools/uni_bench.py [--reps 5] [--shape 40x8388608 640x1048576]
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_1910_05615_b200 import api

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--shape", nargs="+", default=["std", "ref"],
                    help="NCOLSxLEN, or std (p x n of config 4) / ref (16 p x n/8: one refinement call)")
    ap.add_argument("--dist", default="config4", choices=["config4", "normal", "mixed"],
                    help="config4: the columns of the config-4 data (standardisation: X's columns; refinement: "
                         "the 1M-row blocks of its standardised columns); normal: N(0,1); mixed: N(0,1), "
                         "3 N(0,1) + 100 and lognormal columns in turn")
    a = ap.parse_args()
    ctx = api.new_context(0)
    g = torch.Generator(device="cuda").manual_seed(7)
    res = {}
    Xc = None
    if a.dist == "config4":
        from paper_1910_05615_b200 import datagen
        Xc = torch.from_numpy(datagen.make_config(4).X).cuda().t().contiguous()  # (40, 8M)
    n4 = 8_000_000
    for sh in a.shape:
        sh = {"std": f"40x{n4}", "ref": f"640x{n4 // 8}"}.get(sh, sh)
        nc, ln = (int(v) for v in sh.split("x"))
        if Xc is not None:
            p, n = Xc.shape
            med = Xc.median(dim=1, keepdim=True).values
            Zs = (Xc - med) / (Xc - med).abs().median(dim=1, keepdim=True).values
            assert n >= ln, "config4 columns are at most n rows long"
            blocks = Zs[:, : (n // ln) * ln].reshape(p, n // ln, ln).permute(1, 0, 2).reshape(-1, ln)
            reps = (nc + blocks.shape[0] - 1) // blocks.shape[0]
            cols = (Xc if ln == n else torch.cat([blocks] * reps))[:nc].contiguous()
            del Zs, blocks
        else:
            cols = torch.randn(nc, ln, dtype=torch.float64, device="cuda", generator=g)
            if a.dist == "mixed":
                cols[1::3] = cols[1::3] * 3.0 + 100.0
                cols[2::3] = cols[2::3].exp()
        ts = []
        for r in range(a.reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            api.unimcd(cols, ctx=ctx)
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        res[sh] = {"ms": ms, "GBps_one_read": nc * ln * 8 / ms / 1e6}
        print(json.dumps({sh: res[sh]}), flush=True)
        del cols
    api.destroy_context(ctx)


if __name__ == "__main__":
    main()
