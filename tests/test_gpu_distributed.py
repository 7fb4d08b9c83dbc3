"""The sharded fit (rtdetmcd_fit_sharded: one library call per rank) on one GPU.

Ranks here are threads of one process or separate processes, each with its own library context
(stream, workspace, communicator) on cuda:0.  The exchanges go through the library's host
transport (callbacks into ThreadTransport / TorchTransport over gloo) or through NCCL at world 1:
no kernel ever waits on another rank's kernel (B200_PROFILING.md: ranks that spin on each other
must not share a GPU), the library blocks on the host between its phases.  Results must be
bit-identical to the single-context rtdetmcd_fit with the same contiguous blocks (every cross-block
reduction is a fixed-order fold by block id) and within the north-star tolerances of the oracle.
"""
import os
import socket
import tempfile
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fit as ofit  # noqa: E402
from paper_1910_05615_b200 import api, datagen  # noqa: E402
from paper_1910_05615_b200.distributed import (ThreadTransport, TorchTransport, host_context,  # noqa: E402
                                               shard_rows)
from tests._parity import TOL, assert_flags_equal, rel_mu, rel_sigma  # noqa: E402

pytestmark = pytest.mark.gpu

FIELDS = ("loc", "scale", "mu_raw", "sigma_raw", "mu_rew", "sigma_rew", "block_chosen", "start_steps",
          "start_status", "start_logdet")


def _run_threads(X, h, q, world, X_override=None, opts_override=None, **kw):
    n = X.shape[0]
    hub = ThreadTransport.Hub(world)
    out, errs = [None] * world, [None] * world

    def body(r):
        ctx = None
        try:
            a, b, _, _ = shard_rows(n, q, world, r)
            Xl = X[a:b] if X_override is None else X_override(r, X[a:b])
            Xl = torch.from_numpy(np.ascontiguousarray(Xl)).cuda()
            ctx = host_context(0, ThreadTransport(hub, r))
            okw = dict(kw)
            if opts_override:
                okw.update(opts_override(r))
            out[r] = api.fit_sharded(Xl, n, ctx, h=h, q=q, **okw)
        except api.RTDError as e:
            errs[r] = e
        except Exception as e:  # noqa: BLE001
            errs[r] = e
            hub.barrier.abort()
        finally:
            if ctx is not None:
                api.destroy_context(ctx)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in ts]
    [t.join(timeout=900) for t in ts]
    return out, errs


def _assert_identical(res, single):
    for r in res:
        for k in FIELDS:
            assert np.array_equal(getattr(r, k), getattr(single, k)), k
        assert (r.n_weighted, r.n_kept_blocks, r.n_valid_blocks, r.h, r.h_block, r.q) == \
            (single.n_weighted, single.n_kept_blocks, single.n_valid_blocks, single.h, single.h_block, single.q)
    for k in ("flags", "rd2", "weights", "hsubset"):
        cat = torch.cat([getattr(r, k) for r in res]).cpu().numpy()
        assert np.array_equal(cat, getattr(single, k).cpu().numpy()), k


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_equals_single_context(world):
    n, q = 40_000, 8
    d = datagen.make_config(4, n=n)
    h = int(0.75 * n)
    single = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1)
    res, errs = _run_threads(d.X, h, q, world)
    assert not any(errs), errs
    _assert_identical(res, single)


def test_sharded_matches_oracle_with_remainder():
    n, q = 30_007, 4                      # remainder rows on the last rank
    d = datagen.make_config(2, n=n)
    h = int(0.75 * n)
    o = ofit.fit(d.X, h=h, q=q, partition_mode="contiguous")
    res, errs = _run_threads(d.X, h, q, 2)
    assert not any(errs), errs
    for r in res:
        assert rel_sigma(r.sigma_rew, o.Sigma_rew) < TOL
        assert rel_mu(r.mu_rew, o.mu_rew, o.Sigma_rew) < TOL
        assert rel_sigma(r.sigma_raw, o.Sigma_raw) < TOL
    flags = torch.cat([r.flags for r in res]).cpu().numpy()
    rd2 = torch.cat([r.rd2 for r in res]).cpu().numpy()
    assert_flags_equal(flags, o.flags, o.rd2, o.cutoff2)
    assert np.allclose(rd2, o.rd2, rtol=1e-9, atol=1e-9)
    w = torch.cat([r.weights for r in res]).cpu().numpy().astype(bool)
    assert not w[4 * (n // 4):].any()     # remainder rows: flagged, not fitted (reading R23)
    assert int(w.sum()) == res[0].n_weighted


def test_sharded_errors_agree_on_every_rank():
    n, q = 12_000, 4
    d = datagen.make_config(2, n=n)
    h = int(0.75 * n)

    def nan_on_rank1(r, Xl):
        Xl = Xl.copy()
        if r == 1:
            Xl[17, 3] = np.nan
        return Xl

    _, errs = _run_threads(d.X, h, q, 2, X_override=nan_on_rank1)
    assert all(isinstance(e, api.RTDError) and e.name == "RTD_E_NONFINITE" for e in errs), errs
    assert all(f"row {n // 2 + 17}" in str(e) for e in errs)           # global row index on both ranks
    _, errs = _run_threads(d.X, h, q, 2, opts_override=lambda r: {"quantile": 0.975 if r == 0 else 0.99})
    assert all(isinstance(e, api.RTDError) and e.name == "RTD_E_INVALID_ARG" for e in errs), errs
    _, errs = _run_threads(d.X, h, 3, 2)                             # q not a multiple of the world
    assert all(isinstance(e, api.RTDError) and e.name == "RTD_E_INVALID_ARG" for e in errs), errs


def test_sharded_nccl_world1_equals_single_context():
    # the NCCL transport inside the library (all-gathers, grouped send/recv incl. to self) at world 1
    n, q = 40_000, 4
    d = datagen.make_config(4, n=n)
    h = int(0.75 * n)
    single = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1)
    ctx = api.dist_context(0, 0, 1, api.nccl_unique_id())
    try:
        assert api.ctx_comm(ctx) == (0, 1, "nccl")
        r = api.fit_sharded(torch.from_numpy(d.X).cuda(), n, ctx, h=h, q=q)
        rh = api.fit_sharded(d.X, n, ctx, h=h, q=q)                 # host rows: copied by the library
    finally:
        api.destroy_context(ctx)
    _assert_identical([r], single)
    assert np.array_equal(rh.sigma_rew, single.sigma_rew) and np.array_equal(rh.flags, single.flags.cpu().numpy())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _proc_worker(rank, world, port, outdir, n, q, h):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        d = datagen.make_config(4, n=n)
        a, b, _, _ = shard_rows(n, q, world, rank)
        ctx = host_context(0, TorchTransport())
        r = api.fit_sharded(torch.from_numpy(np.ascontiguousarray(d.X[a:b])).cuda(), n, ctx, h=h, q=q)
        np.savez(os.path.join(outdir, f"r{rank}.npz"), flags=r.flags.cpu().numpy(), rd2=r.rd2.cpu().numpy(),
                 weights=r.weights.cpu().numpy(), hsubset=r.hsubset.cpu().numpy(),
                 **{k: getattr(r, k) for k in FIELDS})
        api.destroy_context(ctx)
    finally:
        dist.destroy_process_group()


def test_sharded_two_processes_gloo_transport():
    # two processes (two CUDA contexts on cuda:0), exchanges over gloo through the library's host transport
    import torch.multiprocessing as mp
    n, q = 40_000, 8
    d = datagen.make_config(4, n=n)
    h = int(0.75 * n)
    single = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1)
    with tempfile.TemporaryDirectory() as dd:
        mp.spawn(_proc_worker, args=(2, _free_port(), dd, n, q, h), nprocs=2, join=True)
        z = [np.load(os.path.join(dd, f"r{r}.npz")) for r in range(2)]
    for zr in z:
        for k in FIELDS:
            assert np.array_equal(zr[k], getattr(single, k)), k
    for k in ("flags", "rd2", "weights", "hsubset"):
        assert np.array_equal(np.concatenate([zr[k] for zr in z]), getattr(single, k).cpu().numpy()), k


def test_contiguous_fit_matches_oracle():
    n, q = 24_000, 3
    d = datagen.make_config(4, n=n)
    h = int(0.75 * n)
    o = ofit.fit(d.X, h=h, q=q, partition_mode="contiguous")
    g = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1)
    assert rel_sigma(g.sigma_rew, o.Sigma_rew) < TOL
    assert rel_mu(g.mu_rew, o.mu_rew, o.Sigma_rew) < TOL
    assert_flags_equal(g.flags.cpu().numpy(), o.flags, o.rd2, o.cutoff2)
