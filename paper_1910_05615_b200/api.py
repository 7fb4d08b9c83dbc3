"""Python face of the C ABI (include/rtdetmcd.h): marshalling only.

Inputs may be numpy arrays or torch tensors (CPU or CUDA); the library copies
host buffers itself.  Per-row outputs land on the device of X when X is a
CUDA tensor, else in numpy arrays.  There is no CPU path: every call goes
through libpaper_1910_05615_b200.so and raises if it is missing.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import RTD_STATUS, Opts, Result, Transport, lib


class RTDError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{RTD_STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = RTD_STATUS.get(code, str(code))


def _torch():
    import torch
    return torch


_CTX: dict = {}


def _ctx(device: int = 0):
    """Context per (device, torch current stream)."""
    torch = _torch()
    stream = 0
    if torch.cuda.is_available():
        stream = torch.cuda.current_stream(device).cuda_stream
    key = (device, stream)
    if key not in _CTX:
        h = C.c_void_p()
        rc = lib().rtdetmcd_create(C.byref(h), device, C.c_void_p(stream) if stream else None)
        if rc != 0:
            raise RTDError(rc, "rtdetmcd_create failed")
        _CTX[key] = {"h": h, "ws": None}
    return _CTX[key]


def _sync_torch(device: int) -> None:
    """Make work queued by torch on `device` visible to the library's stream."""
    torch = _torch()
    if torch.cuda.is_available():
        torch.cuda.current_stream(device).synchronize()


def new_context(device: int = 0) -> dict:
    """A private context (own stream, own workspace), e.g. one per rank thread."""
    h = C.c_void_p()
    rc = lib().rtdetmcd_create(C.byref(h), device, None)
    if rc != 0:
        raise RTDError(rc, "rtdetmcd_create failed")
    return {"h": h, "ws": None}


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for rtdetmcd_create_dist (create on one rank, share with the others)."""
    buf = C.create_string_buffer(128)
    rc = lib().rtdetmcd_nccl_unique_id(buf)
    if rc != 0:
        raise RTDError(rc, "rtdetmcd_nccl_unique_id failed (libnccl.so.2 not loadable?)")
    return buf.raw


def dist_context(device: int, rank: int, world: int, unique_id: bytes | None) -> dict:
    """rtdetmcd_create_dist: rank `rank` of `world` over NCCL (collective over the ranks)."""
    h = C.c_void_p()
    idb = C.create_string_buffer(unique_id, 128) if unique_id is not None else None
    rc = lib().rtdetmcd_create_dist(C.byref(h), int(device), None, idb, int(rank), int(world))
    if rc != 0:
        raise RTDError(rc, "rtdetmcd_create_dist failed")
    return {"h": h, "ws": None}


def transport_context(device: int, rank: int, world: int, allgather, alltoallv) -> dict:
    """rtdetmcd_create_transport with Python callbacks on host buffers:
    allgather(send: memoryview, recv: memoryview) and
    alltoallv(send: memoryview, send_bytes, send_offs, recv: memoryview, recv_bytes, recv_offs)."""
    from ._lib import ALLGATHER_FN, ALLTOALLV_FN

    def _ag(user, send, recv, nbytes):
        try:
            allgather((C.c_char * nbytes).from_address(send), (C.c_char * (nbytes * world)).from_address(recv))
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"rtdetmcd transport allgather failed on rank {rank}: {e!r}", flush=True)
            return 1

    def _a2a(user, send, sb, so, recv, rb, ro):
        try:
            sbl, sol = [sb[i] for i in range(world)], [so[i] for i in range(world)]
            rbl, rol = [rb[i] for i in range(world)], [ro[i] for i in range(world)]
            stot = max(a + b for a, b in zip(sol, sbl))
            rtot = max(a + b for a, b in zip(rol, rbl))
            sv = (C.c_char * max(stot, 1)).from_address(send) if send else None
            rv = (C.c_char * max(rtot, 1)).from_address(recv) if recv else None
            alltoallv(sv, sbl, sol, rv, rbl, rol)
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"rtdetmcd transport alltoallv failed on rank {rank}: {e!r}", flush=True)
            return 1

    t = Transport(None, ALLGATHER_FN(_ag), ALLTOALLV_FN(_a2a))
    h = C.c_void_p()
    rc = lib().rtdetmcd_create_transport(C.byref(h), int(device), None, C.byref(t), int(rank), int(world))
    if rc != 0:
        raise RTDError(rc, "rtdetmcd_create_transport failed")
    return {"h": h, "ws": None, "keep": t}   # the callbacks must outlive the context


def destroy_context(ctx: dict) -> None:
    if ctx.get("h"):
        lib().rtdetmcd_destroy(ctx["h"])
        ctx["h"] = None


def ctx_comm(ctx: dict) -> tuple:
    r, w, k = C.c_int32(), C.c_int32(), C.c_char_p()
    _check(lib().rtdetmcd_ctx_comm(ctx["h"], C.byref(r), C.byref(w), C.byref(k)), ctx)
    return r.value, w.value, k.value.decode()


def shard_layout(n_global: int, q: int, world: int, rank: int) -> tuple:
    """(row0, n_local, block0, q_local) of `rank` (rtdetmcd_shard_layout; host arithmetic only)."""
    r0, nl, b0, ql = C.c_int64(), C.c_int64(), C.c_int32(), C.c_int32()
    rc = lib().rtdetmcd_shard_layout(int(n_global), int(q), int(world), int(rank), C.byref(r0), C.byref(nl),
                                     C.byref(b0), C.byref(ql))
    if rc != 0:
        raise RTDError(rc, f"no layout for n={n_global}, q={q}, world={world}, rank={rank}")
    return r0.value, nl.value, b0.value, ql.value


def _error(rc: int, ctx) -> "RTDError | None":
    return RTDError(rc, lib().rtdetmcd_last_error(ctx["h"]).decode()) if rc else None


def _check(rc: int, ctx) -> None:
    if rc != 0:
        raise RTDError(rc, lib().rtdetmcd_last_error(ctx["h"]).decode())


def _as_f64(x):
    """(pointer, keepalive, is_cuda, device) of a C-contiguous float64 buffer."""
    torch = _torch()
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        t = t.contiguous()
        return t.data_ptr(), t, t.is_cuda, (t.device.index or 0) if t.is_cuda else 0
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return a.ctypes.data, a, False, 0


def _out_buffer(n: int, dtype, on_cuda: bool, device: int):
    torch = _torch()
    if on_cuda:
        t = torch.empty(n, dtype={np.uint8: torch.uint8, np.float64: torch.float64}[dtype], device=f"cuda:{device}")
        return t, t.data_ptr()
    a = np.empty(n, dtype=dtype)
    return a, a.ctypes.data


def default_opts(**kw) -> Opts:
    o = Opts()
    lib().rtdetmcd_opts_default(C.byref(o))
    for k, v in kw.items():
        if v is None:
            continue
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, v)
    return o


@dataclass
class Fit:
    loc: np.ndarray
    scale: np.ndarray
    mu_raw: np.ndarray
    sigma_raw: np.ndarray
    mu_rew: np.ndarray
    sigma_rew: np.ndarray
    logdet_raw: float
    cutoff2: float
    h: int
    h_block: int
    m: int
    q: int
    warnings: int
    n_valid_blocks: int
    n_kept_blocks: int
    n_weighted: int
    block_chosen: np.ndarray
    start_steps: np.ndarray
    start_status: np.ndarray
    start_logdet: np.ndarray
    flags: object = None
    rd2: object = None
    weights: object = None
    hsubset: object = None
    extra: dict = field(default_factory=dict)


def workspace_size(n: int, p: int, **opts) -> int:
    o = default_opts(**opts)
    return int(lib().rtdetmcd_fit_workspace_size(n, p, C.byref(o)))


def _result_buffers(n, p, q, outputs, out_buffers, is_cuda, dev):
    """A Result struct with its host arrays and per-row output buffers (caller-provided or new)."""
    r = Result()
    host = {k: np.zeros(p) for k in ("loc", "scale", "mu_raw", "mu_rew")}
    host.update({k: np.zeros((p, p)) for k in ("sigma_raw", "sigma_rew")})
    qmax = int(q) if q and q > 0 else 1024
    host["block_chosen"] = np.zeros(qmax, np.int32)
    host["start_steps"] = np.zeros(2 * qmax, np.int32)
    host["start_status"] = np.zeros(2 * qmax, np.int32)
    host["start_logdet"] = np.zeros(2 * qmax, np.float64)
    for k, a in host.items():
        setattr(r, k, a.ctypes.data)
    rows = {}
    for k, dt in (("flags", np.uint8), ("rd2", np.float64), ("weights", np.uint8), ("hsubset", np.uint8)):
        if out_buffers and k in out_buffers:          # caller-provided buffer (e.g. pinned host tensor)
            buf = out_buffers[k]
            rows[k] = buf
            setattr(r, k, buf.data_ptr() if hasattr(buf, "data_ptr") else buf.ctypes.data)
        elif k in outputs:
            buf, bp = _out_buffer(n, dt, is_cuda, dev)
            rows[k] = buf
            setattr(r, k, bp)
    return r, host, rows


def _make_fit(r, host, rows) -> "Fit":
    qu = r.q_used
    return Fit(loc=host["loc"], scale=host["scale"], mu_raw=host["mu_raw"], sigma_raw=host["sigma_raw"],
               mu_rew=host["mu_rew"], sigma_rew=host["sigma_rew"], logdet_raw=r.logdet_raw, cutoff2=r.cutoff2,
               h=r.h, h_block=r.h_block, m=r.m, q=qu, warnings=r.warnings, n_valid_blocks=r.n_valid_blocks,
               n_kept_blocks=r.n_kept_blocks, n_weighted=r.n_weighted,
               block_chosen=host["block_chosen"][:qu].copy(), start_steps=host["start_steps"][:2 * qu].copy(),
               start_status=host["start_status"][:2 * qu].copy(), start_logdet=host["start_logdet"][:2 * qu].copy(),
               **rows)


def fit(X, h: int | None = None, alpha: float = 0.5, q: int = 1, seed: int = 0, kappa_max: float = 1000.0,
        quantile: float = 0.975, max_csteps: int = 100, refresh_every: int = 32, partition: int = 0,
        log_transform: bool = False, outputs=("flags", "rd2", "weights", "hsubset"), device: int | None = None,
        torch_workspace: bool = True, out_buffers: dict | None = None, ctx: dict | None = None,
        warm_start=None, distance: int = 0, consistency: int = 0) -> Fit:
    """rtdetmcd_fit on an n x p row-major float64 matrix (numpy or torch, host or device).

    warm_start=(mu, sigma): rtdetmcd_fit_warm -- the C-steps of every block start from this
    previous fit (X units, after ln when log_transform) instead of the refined initial estimators.
    distance: RTD_DIST_CHOLESKY (0) | RTD_DIST_INVERSE (1, Table 1 variant I) | RTD_DIST_SMW (2: the
    inverse updated by Sherman-Morrison-Woodbury on single-swap C-steps);
    refresh_every=1 gives the plain-recompute C-steps of variants I / ID.  consistency: RTD_CONS_ALPHA (0) | RTD_CONS_MEDIAN (1).
    """
    ptr, keep, is_cuda, dev = _as_f64(X)
    n, p = int(keep.shape[0]), int(keep.shape[1])
    dev = dev if device is None else device
    ctx = ctx or _ctx(dev)
    if is_cuda:
        _sync_torch(dev)
    o = default_opts(h=int(h or 0), alpha=float(alpha), shards=int(q), seed=int(seed), kappa_max=float(kappa_max),
                     quantile=float(quantile), max_csteps=int(max_csteps), refresh_every=int(refresh_every),
                     partition=int(partition), log_transform=int(bool(log_transform)), distance=int(distance),
                     consistency=int(consistency))
    L = lib()
    if torch_workspace:
        torch = _torch()
        need = int(L.rtdetmcd_fit_workspace_size(n, p, C.byref(o)))
        ws = ctx["ws"]
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{dev}")
            ctx["ws"] = ws
        _check(L.rtdetmcd_set_workspace(ctx["h"], C.c_void_p(ws.data_ptr()), ws.numel()), ctx)
    r, host, rows = _result_buffers(n, p, q, outputs, out_buffers, is_cuda, dev)
    if warm_start is None:
        rc = L.rtdetmcd_fit(ctx["h"], C.c_void_p(ptr), n, p, C.byref(o), C.byref(r))
    else:
        wm = np.ascontiguousarray(warm_start[0], dtype=np.float64).reshape(p)
        wS = np.ascontiguousarray(warm_start[1], dtype=np.float64).reshape(p, p)
        rc = L.rtdetmcd_fit_warm(ctx["h"], C.c_void_p(ptr), n, p, C.byref(o), C.c_void_p(wm.ctypes.data),
                                 C.c_void_p(wS.ctypes.data), C.byref(r))
    err = _error(rc, ctx)          # read before the workspace reset (every library call clears the message)
    if torch_workspace:
        L.rtdetmcd_set_workspace(ctx["h"], None, 0)
    if err:
        raise err
    return _make_fit(r, host, rows)


def fit_sharded(X_local, n_global: int, ctx: dict, h: int | None = None, alpha: float = 0.5, q: int = 0,
                seed: int = 0, kappa_max: float = 1000.0, quantile: float = 0.975, max_csteps: int = 100,
                refresh_every: int = 32, log_transform: bool = False, outputs=("flags", "rd2", "weights", "hsubset"),
                out_buffers: dict | None = None, distance: int = 0, consistency: int = 0) -> Fit:
    """rtdetmcd_fit_sharded (collective): this rank's rows X_local (shard_layout) of an n_global-row data
    set; global estimates, local per-row outputs.  Contiguous blocks (the sharded partition)."""
    ptr, keep, is_cuda, dev = _as_f64(X_local)
    n, p = int(keep.shape[0]), int(keep.shape[1])
    if is_cuda:
        _sync_torch(dev)
    o = default_opts(h=int(h or 0), alpha=float(alpha), shards=int(q), seed=int(seed), kappa_max=float(kappa_max),
                     quantile=float(quantile), max_csteps=int(max_csteps), refresh_every=int(refresh_every),
                     partition=1, log_transform=int(bool(log_transform)), distance=int(distance),
                     consistency=int(consistency))
    r, host, rows = _result_buffers(n, p, q, outputs, out_buffers, is_cuda, dev)
    _check(lib().rtdetmcd_fit_sharded(ctx["h"], C.c_void_p(ptr), n, int(n_global), p, C.byref(o), C.byref(r)), ctx)
    return _make_fit(r, host, rows)


def fit_batches(batches, h: int | None = None, alpha: float = 0.5, q: int = 1, seed: int = 0,
                kappa_max: float = 1000.0, quantile: float = 0.975, max_csteps: int = 100, refresh_every: int = 32,
                partition: int = 0, log_transform: bool = False, outputs=("flags",), out_buffers=None,
                device: int = 0, torch_workspace: bool = True, ctx: dict | None = None, distance: int = 0,
                consistency: int = 0) -> list:
    """rtdetmcd_fit_batches: one fit per HOST batch (n x p row-major float64, pinned torch tensors for
    full overlap), batch b+1's host->device copy overlapping batch b's fit.  out_buffers: None, one
    dict for every batch, or a list of dicts (per batch)."""
    arrs = [_as_f64(X) for X in batches]
    if any(a[2] for a in arrs):
        raise ValueError("fit_batches takes host batches")
    n, p = int(arrs[0][1].shape[0]), int(arrs[0][1].shape[1])
    if any(tuple(a[1].shape) != (n, p) for a in arrs):
        raise ValueError("all batches must have the same shape")
    ctx = ctx or _ctx(device)
    o = default_opts(h=int(h or 0), alpha=float(alpha), shards=int(q), seed=int(seed), kappa_max=float(kappa_max),
                     quantile=float(quantile), max_csteps=int(max_csteps), refresh_every=int(refresh_every),
                     partition=int(partition), log_transform=int(bool(log_transform)), distance=int(distance),
                     consistency=int(consistency))
    L = lib()
    if torch_workspace:
        torch = _torch()
        need = int(L.rtdetmcd_fit_workspace_size(n, p, C.byref(o)))
        ws = ctx["ws"]
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{device}")
            ctx["ws"] = ws
        _check(L.rtdetmcd_set_workspace(ctx["h"], C.c_void_p(ws.data_ptr()), ws.numel()), ctx)
    nb = len(arrs)
    per = []
    for b in range(nb):
        ob = out_buffers[b] if isinstance(out_buffers, (list, tuple)) else out_buffers
        per.append(_result_buffers(n, p, q, outputs, ob, False, device))
    res = (Result * nb)()
    for b in range(nb):
        res[b] = per[b][0]
    ptrs = (C.c_void_p * nb)(*[a[0] for a in arrs])
    rc = L.rtdetmcd_fit_batches(ctx["h"], ptrs, nb, n, p, C.byref(o), res)
    err = _error(rc, ctx)          # read before the workspace reset (every library call clears the message)
    if torch_workspace:
        L.rtdetmcd_set_workspace(ctx["h"], None, 0)
    if err:
        raise err
    return [_make_fit(res[b], per[b][1], per[b][2]) for b in range(nb)]


def flag(X, mu, sigma, quantile: float = 0.975, log_transform: bool = False, want_rd2: bool = True,
         ctx: dict | None = None):
    """rtdetmcd_flag: (flags, rd2) of rows of X under (mu, sigma)."""
    ptr, keep, is_cuda, dev = _as_f64(X)
    n, p = int(keep.shape[0]), int(keep.shape[1])
    ctx = ctx or _ctx(dev)
    if is_cuda:
        _sync_torch(dev)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    sg = np.ascontiguousarray(sigma, dtype=np.float64)
    fl, fp = _out_buffer(n, np.uint8, is_cuda, dev)
    rd, rp = _out_buffer(n, np.float64, is_cuda, dev) if want_rd2 else (None, None)
    _check(lib().rtdetmcd_flag(ctx["h"], C.c_void_p(ptr), n, p, mu.ctypes.data, sg.ctypes.data, float(quantile),
                               int(bool(log_transform)), C.c_void_p(fp), C.c_void_p(rp) if rp else None), ctx)
    return fl, rd


def unimcd(cols, device: int = 0, ctx: dict | None = None):
    """Univariate reweighted MCD of each column of a (ncols, len) device tensor."""
    ptr, keep, is_cuda, dev = _as_f64(cols)
    if not is_cuda:
        raise ValueError("unimcd stage call takes a CUDA tensor (ncols, len)")
    ncols, ln = int(keep.shape[0]), int(keep.shape[1])
    ctx = ctx or _ctx(dev)
    _sync_torch(dev)
    out = {k: np.zeros(ncols) for k in ("loc", "scale", "raw_loc", "raw_var")}
    start = np.zeros(ncols, np.int64)
    _check(lib().rtdetmcd_unimcd(ctx["h"], C.c_void_p(ptr), ln, ncols, out["loc"].ctypes.data,
                                 out["scale"].ctypes.data, out["raw_loc"].ctypes.data, out["raw_var"].ctypes.data,
                                 start.ctypes.data), ctx)
    out["start"] = start
    return out


def _zcols(Z):
    """Z given as a (m, p) CUDA tensor -> column-major device buffer."""
    torch = _torch()
    if not (isinstance(Z, torch.Tensor) and Z.is_cuda):
        raise ValueError("stage calls take a CUDA tensor")
    Zc = Z.detach().to(torch.float64).t().contiguous()
    _sync_torch(Z.device.index or 0)
    return Zc, int(Z.shape[0]), int(Z.shape[1]), Z.device.index or 0


def initial(Z):
    Zc, m, p, dev = _zcols(Z)
    ctx = _ctx(dev)
    S1, S2 = np.zeros((p, p)), np.zeros((p, p))
    ok = C.c_int32()
    _check(lib().rtdetmcd_initial(ctx["h"], C.c_void_p(Zc.data_ptr()), m, p, S1.ctypes.data, S2.ctypes.data,
                                  C.byref(ok)), ctx)
    return S1, S2, bool(ok.value)


def refine(Z, S, kappa_max: float = 1000.0):
    Zc, m, p, dev = _zcols(Z)
    ctx = _ctx(dev)
    S = np.ascontiguousarray(S, dtype=np.float64)
    mu, sg, lam = np.zeros(p), np.zeros((p, p)), np.zeros(p)
    ok = C.c_int32()
    _check(lib().rtdetmcd_refine(ctx["h"], C.c_void_p(Zc.data_ptr()), m, p, S.ctypes.data, float(kappa_max),
                                 mu.ctypes.data, sg.ctypes.data, lam.ctypes.data, C.byref(ok)), ctx)
    return mu, sg, lam, bool(ok.value)


def csteps(Z, mu0, sigma0, h: int, kappa_max: float = 1000.0, max_steps: int = 100, refresh_every: int = 32):
    torch = _torch()
    Zc, m, p, dev = _zcols(Z)
    ctx = _ctx(dev)
    mu0 = np.ascontiguousarray(mu0, dtype=np.float64)
    s0 = np.ascontiguousarray(sigma0, dtype=np.float64)
    mu, sg = np.zeros(p), np.zeros((p, p))
    ld = C.c_double()
    steps, status = C.c_int32(), C.c_int32()
    hs = torch.empty(m, dtype=torch.uint8, device=Zc.device)
    traj = np.full(max_steps + 1, np.nan)
    _check(lib().rtdetmcd_csteps(ctx["h"], C.c_void_p(Zc.data_ptr()), m, p, int(h), mu0.ctypes.data, s0.ctypes.data,
                                 float(kappa_max), int(max_steps), int(refresh_every), mu.ctypes.data, sg.ctypes.data,
                                 C.byref(ld), C.byref(steps), C.byref(status), C.c_void_p(hs.data_ptr()),
                                 traj.ctypes.data), ctx)
    return {"mu": mu, "sigma": sg, "logdet": ld.value, "steps": steps.value, "status": status.value,
            "hsubset": hs, "logdet_traj": traj}


def chi2_quantile(prob: float, dof: int) -> float:
    return float(lib().rtdetmcd_chi2_quantile(float(prob), int(dof)))


def consistency_factor(alpha: float, p: int) -> float:
    return float(lib().rtdetmcd_consistency_factor(float(alpha), int(p)))


def choose_q(n: int, p: int, omega: int = 4096, cap: int = 0) -> int:
    return int(lib().rtdetmcd_choose_q(int(n), int(p), int(omega), int(cap)))


def partition_perm(n: int, seed: int, device: int = 0) -> np.ndarray:
    ctx = _ctx(device)
    out = np.zeros(n, np.int64)
    _check(lib().rtdetmcd_partition_perm(ctx["h"], int(n), C.c_uint64(seed & (2 ** 64 - 1)), out.ctypes.data), ctx)
    return out


def set_profiling(on: bool = True, device: int = 0, ctx: dict | None = None) -> None:
    ctx = ctx or _ctx(device)
    _check(lib().rtdetmcd_set_profiling(ctx["h"], int(bool(on))), ctx)


def profile(device: int = 0, ctx: dict | None = None) -> dict:
    """{kernel class: {"ms", "launches", "bytes" (algorithmic HBM), "flops", "eff_bytes"}} since set_profiling."""
    ctx = ctx or _ctx(device)
    L = lib()
    out = {}
    for i in range(L.rtdetmcd_prof_count(ctx["h"])):
        name = C.create_string_buffer(64)
        ms, n, by, fl, eb = C.c_double(), C.c_int64(), C.c_double(), C.c_double(), C.c_double()
        _check(L.rtdetmcd_prof_entry(ctx["h"], i, name, 64, C.byref(ms), C.byref(n), C.byref(by), C.byref(fl),
                                     C.byref(eb)), ctx)
        out[name.value.decode()] = {"ms": ms.value, "launches": n.value, "bytes": by.value, "flops": fl.value,
                                    "eff_bytes": eb.value}
    return out


def counters() -> tuple:
    """(hand-written kernel launches, CUB sort invocations) issued by the library so far."""
    k, s = C.c_int64(), C.c_int64()
    lib().rtdetmcd_counters(C.byref(k), C.byref(s))
    return k.value, s.value
