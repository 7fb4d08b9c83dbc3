"""An engine with the interface of distributed.GpuEngine whose arithmetic is the CPU oracle.

Test infrastructure: it lets the CPU (gloo / thread) tests drive the real
sharded orchestration (column exchange, record gathers, pooling order) of
paper_1910_05615_b200/distributed.py without a GPU.  The product never uses it.
"""
import math

import numpy as np
import torch

from oracle import fit as ofit
from oracle.chi2 import chi2_quantile, consistency_factor
from oracle.numerics import mahalanobis_sq
from oracle.parallel import select_and_pool
from oracle.unimcd import unimcd_reweighted


class OracleEngine:
    torch = torch

    def __init__(self):
        self.device = torch.device("cpu")

    def columns(self, X_local, log_transform):
        X = X_local.numpy()
        if not np.all(np.isfinite(X)):
            raise ValueError("nonfinite")
        if log_transform:
            X = np.log(X)
        return torch.from_numpy(np.ascontiguousarray(X.T))

    def unimcd(self, cols):
        us = [unimcd_reweighted(c) for c in cols.numpy()]
        return np.array([u.loc for u in us]), np.array([u.scale for u in us])

    def blocks_fit(self, X_blocks, loc, scale, q_local, q_global, h_block, opts):
        X = X_blocks.numpy()
        if opts.log_transform:
            X = np.log(X)
        self.loc, self.scale = np.asarray(loc), np.asarray(scale)
        Z = (X - self.loc) / self.scale
        n, p = Z.shape
        m = n // q_local
        self.blocks = [Z[b * m:(b + 1) * m] for b in range(q_local)]
        self.m, self.p = m, p
        recs = np.zeros((q_local, 4 + p + p * p))
        for b, Zb in enumerate(self.blocks):
            starts, chosen = ofit.fit_block(Zb, h_block, opts.kappa_max, opts.max_csteps)
            if chosen < 0:
                continue
            st = starts[chosen]
            recs[b, :4] = [1.0, chosen, st.logdet, st.steps]
            recs[b, 4:4 + p] = st.mu
            recs[b, 4 + p:] = (consistency_factor(h_block / m, p) * st.Sigma).ravel()
        return recs

    def aggregate(self, q, p, m, records):
        valid = [b for b in range(q) if records[b, 0] != 0]
        mus = [records[b, 4:4 + p] for b in valid]
        Ss = [records[b, 4 + p:].reshape(p, p) for b in valid]
        if q == 1:
            self.mu_raw, self.S_raw, kept = mus[0], Ss[0], [0]
        else:
            self.mu_raw, self.S_raw, kept, _ = select_and_pool(mus, Ss, [m] * len(valid), valid)
        return self.mu_raw, self.S_raw, len(kept)

    def blocks_reweight(self, quantile, q_local, p, nrows):
        c2 = chi2_quantile(quantile, p)
        sums = np.zeros((q_local, p + p * (p + 1) // 2 + 1))
        ws = []
        il = np.tril_indices(p)
        for b, Zb in enumerate(self.blocks):
            w = mahalanobis_sq(Zb, self.mu_raw, self.S_raw) <= c2
            D = Zb[w] - self.mu_raw
            S2 = D.T @ D
            sums[b, :p] = D.sum(0)
            sums[b, p:-1] = S2[il]
            sums[b, -1] = w.sum()
            ws.append(w)
        return sums, torch.from_numpy(np.concatenate(ws).astype(np.uint8))

    def pool_reweight(self, q, sums, quantile, p):
        tot = np.zeros(sums.shape[1])
        for b in range(q):
            tot += sums[b]
        k = tot[-1]
        S1 = tot[:p]
        S2 = np.zeros((p, p))
        il = np.tril_indices(p)
        S2[il] = tot[p:-1]
        S2 = S2 + np.tril(S2, -1).T
        mu_rew = self.mu_raw + S1 / k
        S_rew = consistency_factor(quantile, p) * (S2 - np.outer(S1, S1) / k) / (k - 1)
        ss = np.outer(self.scale, self.scale)
        return {"mu_raw": self.loc + self.scale * self.mu_raw, "sigma_raw": self.S_raw * ss,
                "mu_rew": self.loc + self.scale * mu_rew, "sigma_rew": S_rew * ss, "n_weighted": int(k)}

    def flag(self, X_local, mu, sigma, quantile, log_transform):
        X = X_local.numpy()
        if log_transform:
            X = np.log(X)
        rd2, fl, _ = ofit.flag(X, mu, sigma, quantile)
        return fl.astype(np.uint8), rd2


def dummy_opts(log_transform=False):
    class O:
        pass
    o = O()
    o.kappa_max, o.max_csteps, o.log_transform = 1000.0, 100, int(log_transform)
    return o


def nearly(a, b, tol=1e-10):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)) < tol and math.isfinite(float(np.sum(a)))
