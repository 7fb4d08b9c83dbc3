"""Row-sharded RT-DetMCD, one process (rank) per GPU (§4 steps 1-10).

The whole sharded fit is ONE library call, `rtdetmcd_fit_sharded` (include/rtdetmcd.h): the library
does the column all-to-all of the global standardisation, the all-gathers of block records and of
reweighting sums, and the deterministic folds, over NCCL (`rtdetmcd_create_dist`) or over
caller-supplied host callbacks (`rtdetmcd_create_transport`).  This module is a thin caller: it
makes the context (NCCL unique id shared over torch.distributed, or a host transport over a
torch.distributed group or over threads of one process), slices this rank's rows and calls the
library.  No arithmetic of the method runs here.

Row layout (rtdetmcd_shard_layout): q blocks of m = n // q consecutive rows; rank r holds blocks
[r q/G, (r+1) q/G); the last rank also holds the n - q m remainder rows (flagged, not fitted).
BASELINE.json configs[3]: "rows sharded evenly over 1/2/4/8 GPUs with per-shard DetMCD".
"""
from __future__ import annotations

import threading

import numpy as np

from . import api


def shard_rows(n: int, q: int, world: int, rank: int):
    """(a, b, m, q_local): rows [a, b) of `rank` (rtdetmcd_shard_layout)."""
    row0, n_local, _, q_local = api.shard_layout(n, q, world, rank)
    return row0, row0 + n_local, n // q, q_local


# ------------------------------------------------------------------ host transports (rtdetmcd_transport)
class TorchTransport:
    """Host-buffer collectives over a torch.distributed group (gloo on CPU; works on any backend that
    takes CPU tensors).  all-gather -> dist.all_gather; all-to-all-v -> paired isend / irecv."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _t(self, view, nbytes=None):
        a = np.frombuffer(view, dtype=np.uint8, count=len(view) if nbytes is None else nbytes)
        return self.torch.from_numpy(a)

    def allgather(self, send, recv):
        nb = len(send)
        src = self._t(send).clone()
        outs = [self.torch.empty(nb, dtype=self.torch.uint8) for _ in range(self.world)]
        self.dist.all_gather(outs, src, group=self.group)
        dst = np.frombuffer(recv, dtype=np.uint8)
        for r in range(self.world):
            dst[r * nb:(r + 1) * nb] = outs[r].numpy()

    def alltoallv(self, send, sb, so, recv, rb, ro):
        torch = self.torch
        sbuf = np.frombuffer(send, dtype=np.uint8) if send is not None else np.zeros(0, np.uint8)
        rbuf = np.frombuffer(recv, dtype=np.uint8) if recv is not None else np.zeros(0, np.uint8)
        reqs, tmp = [], {}
        for s in range(self.world):
            if s == self.rank:
                rbuf[ro[s]:ro[s] + rb[s]] = sbuf[so[s]:so[s] + sb[s]]
                continue
            if sb[s]:
                t = torch.from_numpy(sbuf[so[s]:so[s] + sb[s]].copy())
                tmp[("s", s)] = t
                reqs.append(self.dist.isend(t, self._g(s), group=self.group))
            if rb[s]:
                t = torch.empty(rb[s], dtype=torch.uint8)
                tmp[("r", s)] = t
                reqs.append(self.dist.irecv(t, self._g(s), group=self.group))
        for q in reqs:
            q.wait()
        for s in range(self.world):
            if s != self.rank and rb[s]:
                rbuf[ro[s]:ro[s] + rb[s]] = tmp[("r", s)].numpy()

    def _g(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)


class ThreadTransport:
    """Ranks as threads of one process (one object per rank, sharing a Hub)."""

    class Hub:
        def __init__(self, world):
            self.world = world
            self.barrier = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, hub: "ThreadTransport.Hub", rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def _exchange(self, obj):
        self.hub.barrier.wait()
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()
        got = list(self.hub.slots)
        self.hub.barrier.wait()
        return got

    def allgather(self, send, recv):
        nb = len(send)
        got = self._exchange(bytes(send))
        dst = np.frombuffer(recv, dtype=np.uint8)
        for r, g in enumerate(got):
            dst[r * nb:(r + 1) * nb] = np.frombuffer(g, dtype=np.uint8)

    def alltoallv(self, send, sb, so, recv, rb, ro):
        src = np.frombuffer(send, dtype=np.uint8) if send is not None else np.zeros(0, np.uint8)
        got = self._exchange([src[so[s]:so[s] + sb[s]].copy() for s in range(self.world)])
        dst = np.frombuffer(recv, dtype=np.uint8) if recv is not None else np.zeros(0, np.uint8)
        for s in range(self.world):
            part = got[s][self.rank]
            assert part.size == rb[s], (part.size, rb[s])
            dst[ro[s]:ro[s] + rb[s]] = part


def host_context(device: int, transport) -> dict:
    """A library context over a host transport (TorchTransport / ThreadTransport)."""
    return api.transport_context(device, transport.rank, transport.world, transport.allgather, transport.alltoallv)


def nccl_context(device: int, group=None) -> dict:
    """A library context over NCCL: rank 0 of the torch.distributed group makes the unique id, the
    group broadcasts it (plumbing), every rank creates its communicator inside the library."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    box = [api.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0 if group is None else dist.get_global_rank(group, 0), group=group)
    return api.dist_context(device, rank, world, box[0])


class ShardedFit:
    """bench.py helper: this rank's rows of a dataset on its GPU (or pinned host memory), one `step()` =
    one rtdetmcd_fit_sharded (fit + flag of the local rows) over NCCL."""

    def __init__(self, X, h, q, log_transform, rank, world, device, host=False):
        import torch
        n = X.shape[0]
        a, b, _, _ = shard_rows(n, q, world, rank)
        self.n, self.h, self.q, self.log = n, h, q, log_transform
        Xl = torch.from_numpy(np.ascontiguousarray(X[a:b]))
        self.X_local = Xl.pin_memory() if host else Xl.to(f"cuda:{device}")
        self.n_local = b - a
        self.ctx = nccl_context(device)
        fl = torch.empty(self.n_local, dtype=torch.uint8)
        self.flags = fl.pin_memory() if host else fl.to(f"cuda:{device}")

    def step(self):
        return api.fit_sharded(self.X_local, self.n, self.ctx, h=self.h, q=self.q, log_transform=self.log,
                               outputs=(), out_buffers={"flags": self.flags})
