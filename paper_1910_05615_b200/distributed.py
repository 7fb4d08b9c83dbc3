"""Row-sharded RT-DetMCD: one process (or rank) per GPU (§4 steps 1-10).

Rank r holds the contiguous rows of blocks [r q/G, (r+1) q/G) (BASELINE.json
configs[3]: "rows sharded evenly over 1/2/4/8 GPUs with per-shard DetMCD";
the last rank also holds the n - q m remainder rows, which are flagged but not
fitted).  The exchange points are exactly the method's couplings:

  1. global standardisation: column all-to-all, the owner
     of column j runs the univariate MCD over all n rows, loc/scale all-gathered;
  2. block fits (steps 1-4) are rank-local;
  3. aggregation (steps 5-7): the per-block records are all-gathered in block
     order and every rank runs the same deterministic median / KL / pooling;
  4. reweighting (steps 8-9): per-block sums all-gathered, pooled in block order;
  5. flagging (step 10) is rank-local.

All arithmetic runs in the engine (GpuEngine = the C ABI of
libpaper_1910_05615_b200.so); this module only moves data.  `comm` is
TorchComm (torch.distributed: NCCL on GPUs, gloo on CPU) or ThreadComm
(ranks as threads of one process, used by the tests).
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass

import numpy as np

from . import api
from ._lib import lib


def record_doubles(p: int) -> int:
    return 4 + p + p * p


# ------------------------------------------------------------------ communication
class TorchComm:
    """torch.distributed collectives on tensors of the engine's device."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather(self, t):
        out = [t.new_empty(t.shape) for _ in range(self.world)]
        self.dist.all_gather(out, t.contiguous(), group=self.group)
        return out

    def all_to_all(self, send, recv_shapes):
        recv = [send[0].new_empty(s) for s in recv_shapes]
        if self.dist.get_backend(self.group) != "gloo":
            self.dist.all_to_all(recv, [x.contiguous() for x in send], group=self.group)
            return recv
        # gloo has no all_to_all: all-gather every rank's padded send list and keep our part
        L = max(int(x.numel()) for x in send) if send else 0
        Lmax = torch_max(self.dist, self.group, L, send[0])
        buf = send[0].new_zeros((self.world, Lmax))
        for s, x in enumerate(send):
            buf[s, :x.numel()] = x.reshape(-1)
        got = self.all_gather(buf)
        return [got[s][self.rank, :int(np.prod(recv_shapes[s]))].reshape(recv_shapes[s]) for s in range(self.world)]


def torch_max(dist, group, value: int, like):
    t = like.new_tensor([float(value)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


class ThreadComm:
    """Collectives between threads of one process (one ThreadComm object per rank, sharing `hub`)."""

    class Hub:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, hub: "ThreadComm.Hub", rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def _exchange(self, obj):
        self.hub.barrier.wait()
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()
        got = list(self.hub.slots)
        self.hub.barrier.wait()
        return got

    def all_gather(self, t):
        return [x.clone() for x in self._exchange(t)]

    def all_to_all(self, send, recv_shapes):
        got = self._exchange(send)
        return [got[s][self.rank].clone().to(send[0].device) for s in range(self.world)]


# ------------------------------------------------------------------ engine: the C ABI
class GpuEngine:
    def __init__(self, device: int = 0):
        import torch
        self.torch = torch
        self.device = torch.device(f"cuda:{device}")
        self.dev_index = device
        self.ctx = api.new_context(device)  # own stream and workspace: the block session lives here

    def _check(self, rc):
        api._check(rc, self.ctx)

    def columns(self, X_local, log_transform: bool):
        torch = self.torch
        api._sync_torch(self.dev_index)
        n, p = X_local.shape
        Xc = torch.empty((p, n), dtype=torch.float64, device=self.device)
        self._check(lib().rtdetmcd_columns(self.ctx["h"], C.c_void_p(X_local.data_ptr()), n, p, int(log_transform),
                                           C.c_void_p(Xc.data_ptr())))
        return Xc

    def unimcd(self, cols):
        r = api.unimcd(cols, device=self.dev_index, ctx=self.ctx)
        return r["loc"], r["scale"]

    def blocks_fit(self, X_blocks, loc, scale, q_local, q_global, h_block, opts):
        n, p = X_blocks.shape
        api._sync_torch(self.dev_index)
        rec = np.zeros((q_local, record_doubles(p)))
        loc = np.ascontiguousarray(loc, dtype=np.float64)
        scale = np.ascontiguousarray(scale, dtype=np.float64)
        self._check(lib().rtdetmcd_blocks_fit(self.ctx["h"], C.c_void_p(X_blocks.data_ptr()), n, p, loc.ctypes.data,
                                              scale.ctypes.data, q_local, q_global, int(h_block), C.byref(opts),
                                              rec.ctypes.data))
        return rec

    def aggregate(self, q, p, m, records):
        records = np.ascontiguousarray(records, dtype=np.float64)
        mu, sg = np.zeros(p), np.zeros((p, p))
        nk = C.c_int32()
        self._check(lib().rtdetmcd_aggregate(self.ctx["h"], q, p, int(m), records.ctypes.data, mu.ctypes.data,
                                             sg.ctypes.data, C.byref(nk)))
        return mu, sg, nk.value

    def blocks_reweight(self, quantile, q_local, p, n_blocks_rows):
        np_ = lib().rtdetmcd_moment_doubles(p)
        sums = np.zeros((q_local, np_))
        w = self.torch.empty(n_blocks_rows, dtype=self.torch.uint8, device=self.device)
        self._check(lib().rtdetmcd_blocks_reweight(self.ctx["h"], float(quantile), sums.ctypes.data,
                                                   C.c_void_p(w.data_ptr())))
        return sums, w

    def pool_reweight(self, q, sums, quantile, p):
        sums = np.ascontiguousarray(sums, dtype=np.float64)
        out = {k: np.zeros(p) for k in ("mu_raw", "mu_rew")}
        out.update({k: np.zeros((p, p)) for k in ("sigma_raw", "sigma_rew")})
        nw = C.c_int64()
        self._check(lib().rtdetmcd_pool_reweight(self.ctx["h"], q, sums.ctypes.data, float(quantile),
                                                 out["mu_raw"].ctypes.data, out["sigma_raw"].ctypes.data,
                                                 out["mu_rew"].ctypes.data, out["sigma_rew"].ctypes.data,
                                                 C.byref(nw)))
        out["n_weighted"] = nw.value
        return out

    def flag(self, X_local, mu, sigma, quantile, log_transform):
        return api.flag(X_local, mu, sigma, quantile=quantile, log_transform=log_transform, ctx=self.ctx)


# ------------------------------------------------------------------ the sharded fit
@dataclass
class ShardResult:
    loc: np.ndarray
    scale: np.ndarray
    mu_raw: np.ndarray
    sigma_raw: np.ndarray
    mu_rew: np.ndarray
    sigma_rew: np.ndarray
    n_kept_blocks: int
    n_weighted: int
    records: np.ndarray        # all blocks, block order
    flags: object              # local rows
    rd2: object
    weights: object            # local block rows (remainder rows: not fitted)


def shard_rows(n: int, q: int, world: int, rank: int):
    """Row range [a, b) of `rank`: blocks [r q/G, (r+1) q/G) of m = n // q rows; the last rank also gets the remainder."""
    if q % world:
        raise ValueError("the number of blocks q must be a multiple of the number of ranks")
    m = n // q
    qb = q // world
    a = rank * qb * m
    b = (rank + 1) * qb * m if rank < world - 1 else n
    return a, b, m, qb


def sharded_fit(X_local, n: int, h: int, q: int, comm, engine, quantile: float = 0.975, kappa_max: float = 1000.0,
                max_csteps: int = 100, refresh_every: int = 32, log_transform: bool = False) -> ShardResult:
    """RT-DetMCD over all ranks; X_local = this rank's rows (shard_rows) on engine.device."""
    torch = engine.torch if hasattr(engine, "torch") else __import__("torch")
    rank, world = comm.rank, comm.world
    n_local, p = int(X_local.shape[0]), int(X_local.shape[1])
    a, b, m, q_local = shard_rows(n, q, world, rank)
    if b - a != n_local:
        raise ValueError(f"rank {rank} expected rows [{a}, {b})")
    dev = engine.device
    # 1. global standardisation: column all-to-all, univariate MCD by the owner, all-gather
    Xc = engine.columns(X_local, log_transform)                     # (p, n_local)
    cpr = math.ceil(p / world)
    counts = [shard_rows(n, q, world, s)[1] - shard_rows(n, q, world, s)[0] for s in range(world)]
    own = [j for j in range(rank * cpr, min(p, (rank + 1) * cpr))]
    full = torch.empty((len(own), n), dtype=torch.float64, device=dev)
    for jj in range(cpr):
        send = []
        for s in range(world):
            j = s * cpr + jj
            send.append(Xc[j] if j < p else Xc.new_empty(0))
        mine = rank * cpr + jj
        shapes = [(counts[s],) if mine < p else (0,) for s in range(world)]
        recv = comm.all_to_all(send, shapes)
        if mine < p:
            off = 0
            for s in range(world):
                full[jj, off:off + counts[s]] = recv[s]
                off += counts[s]
    ls = np.zeros((2, cpr))
    if own:
        loc_o, scale_o = engine.unimcd(full)
        ls[0, :len(own)], ls[1, :len(own)] = loc_o, scale_o
    gathered = comm.all_gather(torch.from_numpy(ls).to(dev))
    loc = np.concatenate([g.cpu().numpy()[0] for g in gathered])[:p]
    scale = np.concatenate([g.cpu().numpy()[1] for g in gathered])[:p]
    # 2. rank-local block fits
    opts = api.default_opts(kappa_max=float(kappa_max), quantile=float(quantile), max_csteps=int(max_csteps),
                            refresh_every=int(refresh_every), log_transform=int(bool(log_transform)))
    h_block = (h * m) // n
    rec = engine.blocks_fit(X_local[: q_local * m], loc, scale, q_local, q, h_block, opts)
    # 3. aggregation on every rank
    all_rec = torch.cat(comm.all_gather(torch.from_numpy(rec).to(dev))).cpu().numpy()
    mu_raw, sigma_raw, n_kept = engine.aggregate(q, p, m, all_rec)
    # 4. distributed reweighting
    sums, weights = engine.blocks_reweight(quantile, q_local, p, q_local * m)
    all_sums = torch.cat(comm.all_gather(torch.from_numpy(sums).to(dev))).cpu().numpy()
    pooled = engine.pool_reweight(q, all_sums, quantile, p)
    # 5. flag the local rows
    flags, rd2 = engine.flag(X_local, pooled["mu_rew"], pooled["sigma_rew"], quantile, log_transform)
    return ShardResult(loc=loc, scale=scale, mu_raw=pooled["mu_raw"], sigma_raw=pooled["sigma_raw"],
                       mu_rew=pooled["mu_rew"], sigma_rew=pooled["sigma_rew"], n_kept_blocks=n_kept,
                       n_weighted=pooled["n_weighted"], records=all_rec, flags=flags, rd2=rd2, weights=weights)


class ShardedFit:
    """bench.py helper: this rank's rows of a dataset, one `step()` = one sharded fit + flag."""

    def __init__(self, X, h, q, seed, log_transform, rank, world, device):
        import torch
        n = X.shape[0]
        a, b, _, _ = shard_rows(n, q, world, rank)
        self.n, self.h, self.q, self.log = n, h, q, log_transform
        self.X_local = torch.from_numpy(np.ascontiguousarray(X[a:b])).to(f"cuda:{device}")
        self.engine = GpuEngine(device)
        self.comm = TorchComm()

    def step(self):
        return sharded_fit(self.X_local, self.n, self.h, self.q, self.comm, self.engine,
                           log_transform=self.log)
