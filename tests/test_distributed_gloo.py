"""The N > 1 plumbing on CPU (no GPU): world_size-2 torch.distributed (gloo) processes and thread ranks.

The sharded fit itself is one library call (rtdetmcd_fit_sharded, exercised on the GPU by
tests/test_gpu_distributed.py).  What runs without a GPU, and is checked here:
  * the row layout of the shards (rtdetmcd_shard_layout: host arithmetic in the library) -- the
    blocks of PAPER.md:750-755 taken contiguously, rank r holding blocks [r q/G, (r+1) q/G), the
    remainder rows (reading R23) on the last rank;
  * the host transports the library calls back into (rtdetmcd_transport): TorchTransport over a
    gloo group of 2 and 3 processes, and ThreadTransport over thread ranks -- all-gather in rank
    order and all-to-all-v with the column-exchange pattern of the global standardisation (C2,
    PAPER.md:756-766): every owner receives its columns' slices from every rank, in rank order.
"""
import os
import socket
import tempfile
import threading

import numpy as np
import pytest

from paper_1910_05615_b200 import api
from paper_1910_05615_b200._lib import RTD_STATUS
from paper_1910_05615_b200.distributed import ThreadTransport, TorchTransport, shard_rows


def test_shard_layout():
    assert shard_rows(10, 4, 2, 0) == (0, 4, 2, 2)
    assert shard_rows(10, 4, 2, 1) == (4, 10, 2, 2)   # last rank keeps the remainder rows
    for n, q, w in [(8_000_000, 8, 1), (8_000_000, 8, 2), (8_000_000, 8, 8), (30_007, 4, 2), (1_001, 6, 3)]:
        spans = [shard_rows(n, q, w, r) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a0, b0, m, ql), (a1, _, _, _) in zip(spans, spans[1:]):
            assert b0 == a1 and ql == q // w and b0 - a0 == ql * m
        assert api.shard_layout(n, q, w, w - 1)[2] == (w - 1) * (q // w)   # block0
    for bad in [(10, 3, 2, 0), (10, 4, 2, 2), (3, 4, 1, 0), (10, 0, 1, 0)]:
        with pytest.raises(api.RTDError) as e:
            api.shard_layout(*bad)
        assert e.value.name == "RTD_E_INVALID_ARG"
    assert RTD_STATUS[10] == "RTD_E_NCCL"


def _column_pattern(world, rank, p, nls):
    """The library's C2 exchange on host buffers: local column-major (p, n_local) -> owned full columns."""
    n_local = nls[rank]
    row0 = sum(nls[:rank])
    cols = np.arange(p)[:, None] * 1_000_000 + (row0 + np.arange(n_local))[None, :]   # value = col*1e6 + global row
    send = np.ascontiguousarray(cols, dtype=np.float64)
    cpr = -(-p // world)
    own0 = min(p, rank * cpr)
    nown = min(p, own0 + cpr) - own0
    sb, so, rb, ro = [], [], [], []
    off = 0
    for s in range(world):
        a0 = min(p, s * cpr)
        cnt = min(p, a0 + cpr) - a0
        sb.append(cnt * n_local * 8)
        so.append(a0 * n_local * 8)
        rb.append(nown * nls[s] * 8)
        ro.append(off)
        off += rb[-1]
    recv = np.zeros(max(off, 8) // 8)
    return send, sb, so, recv, rb, ro, own0, nown


def _exercise(t, p=5, nls=(7, 9, 4)):
    world, rank = t.world, t.rank
    nls = list(nls[:world])
    # all-gather in rank order
    mine = np.full(6, 10.0 * rank + 1.0)
    got = np.zeros(6 * world)
    t.allgather(memoryview(mine).cast("B"), memoryview(got).cast("B"))
    assert np.array_equal(got.reshape(world, 6)[:, 0], 10.0 * np.arange(world) + 1.0)
    # all-to-all-v, column exchange
    send, sb, so, recv, rb, ro, own0, nown = _column_pattern(world, rank, p, nls)
    t.alltoallv(memoryview(send).cast("B"), sb, so, memoryview(recv).cast("B"), rb, ro)
    n = sum(nls)
    full = np.zeros((nown, n))
    for s in range(world):
        part = recv[ro[s] // 8: (ro[s] + rb[s]) // 8].reshape(nown, nls[s])
        full[:, sum(nls[:s]): sum(nls[:s + 1])] = part
    expect = np.arange(own0, own0 + nown)[:, None] * 1_000_000 + np.arange(n)[None, :]
    assert np.array_equal(full, expect)
    return True


@pytest.mark.parametrize("world", [1, 2, 3])
def test_thread_transport(world):
    hub = ThreadTransport.Hub(world)
    ok, errs = [False] * world, []

    def body(r):
        try:
            ok[r] = _exercise(ThreadTransport(hub, r))
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in ts]
    [t.join(timeout=120) for t in ts]
    assert not errs, errs
    assert all(ok)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gloo_worker(rank, world, port, outdir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        _exercise(TorchTransport())
        open(os.path.join(outdir, f"ok{rank}"), "w").write("ok")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_transport_processes(world):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(world, _free_port(), d), nprocs=world, join=True)
        assert all(os.path.exists(os.path.join(d, f"ok{r}")) for r in range(world))
