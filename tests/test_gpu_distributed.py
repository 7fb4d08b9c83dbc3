"""The sharded (N > 1) path with the real CUDA engine: ranks as threads of one process on cuda:0.

Each rank has its own library context (stream, workspace, block session); the
collectives are host-level (ThreadComm), so no kernel waits on another rank's
kernel.  Results must be bit-identical to the single-context fit with the same
contiguous blocks (every cross-block reduction is a fixed-order fold by block
id) and within the north-star tolerances of the oracle.
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fit as ofit  # noqa: E402
from paper_1910_05615_b200 import api, datagen  # noqa: E402
from paper_1910_05615_b200.distributed import GpuEngine, ThreadComm, shard_rows, sharded_fit  # noqa: E402
from tests._parity import TOL, assert_flags_equal, rel_mu, rel_sigma  # noqa: E402

pytestmark = pytest.mark.gpu


def _sharded(X, h, q, world, log=False):
    n = X.shape[0]
    hub = ThreadComm.Hub(world)
    out, errs = [None] * world, []

    def body(r):
        try:
            a, b, _, _ = shard_rows(n, q, world, r)
            Xl = torch.from_numpy(np.ascontiguousarray(X[a:b])).cuda()
            out[r] = sharded_fit(Xl, n, h, q, ThreadComm(hub, r), GpuEngine(0), log_transform=log)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    [t.start() for t in ts]
    [t.join(timeout=900) for t in ts]
    assert not errs, errs
    return out


@pytest.mark.parametrize("world", [1, 2, 4])
def test_sharded_equals_single_context(world):
    n, q = 40_000, 8
    d = datagen.make_config(4, n=n)
    h = int(0.75 * n)
    single = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1)
    res = _sharded(d.X, h, q, world)
    for r in res:
        assert np.array_equal(r.sigma_rew, single.sigma_rew)
        assert np.array_equal(r.mu_rew, single.mu_rew)
        assert np.array_equal(r.sigma_raw, single.sigma_raw)
        assert np.array_equal(r.loc, single.loc) and np.array_equal(r.scale, single.scale)
    flags = torch.cat([r.flags for r in res]).cpu().numpy()
    assert np.array_equal(flags, single.flags.cpu().numpy())


def test_sharded_matches_oracle_with_remainder():
    n, q = 30_007, 4                      # remainder rows on the last rank
    d = datagen.make_config(2, n=n)
    h = int(0.75 * n)
    o = ofit.fit(d.X, h=h, q=q, partition_mode="contiguous")
    res = _sharded(d.X, h, q, 2)
    for r in res:
        assert rel_sigma(r.sigma_rew, o.Sigma_rew) < TOL
        assert rel_mu(r.mu_rew, o.mu_rew, o.Sigma_rew) < TOL
        assert rel_sigma(r.sigma_raw, o.Sigma_raw) < TOL
    flags = torch.cat([r.flags for r in res]).cpu().numpy()
    rd2 = torch.cat([r.rd2 for r in res]).cpu().numpy()
    assert_flags_equal(flags, o.flags, o.rd2, o.cutoff2)
    assert np.allclose(rd2, o.rd2, rtol=1e-9, atol=1e-9)


def test_contiguous_fit_matches_oracle():
    n, q = 24_000, 3
    d = datagen.make_config(4, n=n)
    h = int(0.75 * n)
    o = ofit.fit(d.X, h=h, q=q, partition_mode="contiguous")
    g = api.fit(torch.from_numpy(d.X).cuda(), h=h, q=q, partition=1)
    assert rel_sigma(g.sigma_rew, o.Sigma_rew) < TOL
    assert rel_mu(g.mu_rew, o.mu_rew, o.Sigma_rew) < TOL
    assert_flags_equal(g.flags.cpu().numpy(), o.flags, o.rd2, o.cutoff2)
