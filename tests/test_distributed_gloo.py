"""The N > 1 path on CPU: world_size-2 torch.distributed (gloo) and in-process thread ranks.

The real orchestration of paper_1910_05615_b200/distributed.py (column
all-to-all for the global standardisation, all-gathers of block records and
reweighting sums in block order) runs with an oracle-backed engine; the result
must equal the single-process oracle fit with the same contiguous blocks.
"""
import os
import socket
import tempfile
import threading

import numpy as np
import pytest
import torch

from oracle import fit as ofit
from paper_1910_05615_b200 import datagen
from paper_1910_05615_b200.distributed import ThreadComm, TorchComm, shard_rows, sharded_fit
from tests._oracle_engine import OracleEngine
from tests._parity import rel_mu, rel_sigma

N, Q, CFG = 8_003, 4, 2


def _data():
    d = datagen.make_config(CFG, n=N)
    return d.X, int(0.75 * N)


def _reference():
    X, h = _data()
    return ofit.fit(X, h=h, q=Q, partition_mode="contiguous")


def _check(res_list, ref):
    for r in res_list:
        assert rel_sigma(r["sigma_rew"], ref.Sigma_rew) < 1e-10
        assert rel_mu(r["mu_rew"], ref.mu_rew, ref.Sigma_rew) < 1e-10
        assert rel_sigma(r["sigma_raw"], ref.Sigma_raw) < 1e-10
        assert rel_mu(r["mu_raw"], ref.mu_raw, ref.Sigma_raw) < 1e-10
        assert np.allclose(r["loc"], ref.loc, rtol=1e-14, atol=1e-14)
    flags = np.concatenate([r["flags"] for r in res_list]).astype(bool)
    assert (flags == ref.flags).mean() > 0.9999


def _run_rank(rank, world, comm):
    X, h = _data()
    a, b, _, _ = shard_rows(N, Q, world, rank)
    res = sharded_fit(torch.from_numpy(np.ascontiguousarray(X[a:b])), N, h, Q, comm, OracleEngine())
    return {"sigma_rew": res.sigma_rew, "mu_rew": res.mu_rew, "sigma_raw": res.sigma_raw, "mu_raw": res.mu_raw,
            "loc": res.loc, "flags": np.asarray(res.flags)}


@pytest.mark.parametrize("world", [1, 2, 4])
def test_thread_ranks_match_single_process(world):
    ref = _reference()
    hub = ThreadComm.Hub(world)
    out = [None] * world
    errs = []

    def body(r):
        try:
            out[r] = _run_rank(r, world, ThreadComm(hub, r))
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in ts]
    [t.join(timeout=600) for t in ts]
    assert not errs, errs
    _check(out, ref)


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
        r = _run_rank(rank, world, TorchComm())
        np.savez(os.path.join(outdir, f"r{rank}.npz"), **r)
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2():
    import torch.multiprocessing as mp
    ref = _reference()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_gloo_worker, args=(2, _free_port(), d), nprocs=2, join=True)
        res = []
        for r in range(2):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            res.append({k: z[k] for k in z.files})
    _check(res, ref)


def test_shard_rows():
    assert shard_rows(10, 4, 2, 0) == (0, 4, 2, 2)
    assert shard_rows(10, 4, 2, 1) == (4, 10, 2, 2)   # last rank keeps the remainder rows
    with pytest.raises(ValueError):
        shard_rows(10, 3, 2, 0)
