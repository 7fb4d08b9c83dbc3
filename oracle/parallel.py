"""Partition and robust aggregation of block fits (oracle; test infrastructure only).

PAPER.md:750-755 (§4): randomly partition X into q disjoint blocks of
  m = floor(n/q) cases, discarding the remainder (for fitting).
  Reading R13: the random partition is a keyed Feistel permutation pi of
  [0, n) (6 rounds, cycle-walking, splitmix64 round function); block
  l = {i : floor(pi(i)/m) = l}, position in block = pi(i) - l m.  The same
  counter-based map is implemented independently on the CUDA side.
PAPER.md:1394-1403 (eq. partitionsize): q = max(floor(n/(p omega)), 1), capped.
PAPER.md:860-875 (§4 step 5): entrywise median of the q fits (R14: even q ->
  mean of the two middle values).
PAPER.md:892-898 (eq. KL): KL[(a,A),(b,B)] = tr(A B^-1) - p - log det(A B^-1)
  + (a-b)^T B^-1 (a-b).
PAPER.md:920-974 (§4 steps 6-7): keep the ceil(q/2) fits with lowest KL, then
  single-pass pooling with weight m (eqs. covpool); Sigma_raw = Lambda/(n-1).
"""
from __future__ import annotations

import math

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def choose_q(n: int, p: int, omega: int = 4096, cap: int | None = None) -> int:
    """eq. partitionsize, bounded above by `cap`."""
    q = max(n // (p * omega), 1)
    if cap is not None:
        q = min(q, max(cap, 1))
    return q


def _splitmix64(z: int) -> int:
    z = (z + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _feistel_params(n: int):
    bits = max(2, (n - 1).bit_length())
    bits += bits & 1
    return bits // 2


def feistel_encrypt(x: int, seed: int, half: int) -> int:
    mask = (1 << half) - 1
    L, R = x >> half, x & mask
    for r in range(6):
        F = _splitmix64((seed ^ ((r * GOLDEN) & M64) ^ R) & M64) & mask
        L, R = R, L ^ F
    return (L << half) | R


def feistel_perm(i: int, n: int, seed: int) -> int:
    """pi(i) in [0, n) by cycle-walking the Feistel cipher (reading R13)."""
    half = _feistel_params(n)
    x = feistel_encrypt(i, seed, half)
    while x >= n:
        x = feistel_encrypt(x, seed, half)
    return x


def feistel_perm_array(n: int, seed: int) -> np.ndarray:
    """pi(i) for all i in [0, n): the same map as `feistel_perm`, vectorised (uint64 wraps mod 2^64)."""
    half = _feistel_params(n)
    mask = np.uint64((1 << half) - 1)
    sh = np.uint64(half)
    seed64 = np.uint64(seed & M64)
    rk = [np.uint64((r * GOLDEN) & M64) for r in range(6)]
    c1, c2, c3 = np.uint64(GOLDEN), np.uint64(0xBF58476D1CE4E5B9), np.uint64(0x94D049BB133111EB)

    def enc(x):
        L, R = x >> sh, x & mask
        for r in range(6):
            z = seed64 ^ rk[r] ^ R
            z = z + c1
            z = (z ^ (z >> np.uint64(30))) * c2
            z = (z ^ (z >> np.uint64(27))) * c3
            z = z ^ (z >> np.uint64(31))
            L, R = R, L ^ (z & mask)
        return (L << sh) | R

    with np.errstate(over="ignore"):
        x = enc(np.arange(n, dtype=np.uint64))
        bad = x >= np.uint64(n)
        while bad.any():
            x[bad] = enc(x[bad])
            bad = x >= np.uint64(n)
    return x.astype(np.int64)


def partition(n: int, q: int, seed: int, mode: str = "permute"):
    """(block[i], pos[i], m) for every row; block = -1 for the discarded remainder.

    mode "permute": the keyed random permutation (reading R13);
    mode "contiguous": block l = rows [l m, (l+1) m) (BASELINE.json configs[3]:
    rows sharded over GPUs with per-shard DetMCD).
    """
    m = n // q
    block = np.full(n, -1, dtype=np.int64)
    pos = np.full(n, -1, dtype=np.int64)
    if mode == "contiguous":
        idx = np.arange(q * m)
        block[: q * m] = idx // m
        pos[: q * m] = idx % m
        return block, pos, m
    if q == 1:
        block[:] = 0
        pos[:] = np.arange(n)
        return block, pos, m
    t = feistel_perm_array(n, seed)
    ok = t < q * m
    block[ok] = t[ok] // m
    pos[ok] = t[ok] - block[ok] * m
    return block, pos, m


def block_rows(block: np.ndarray, pos: np.ndarray, l: int, m: int) -> np.ndarray:
    """Original row indices of block l, ordered by position in the block."""
    idx = np.nonzero(block == l)[0]
    out = np.empty(m, dtype=np.int64)
    out[pos[idx]] = idx
    return out


def entrywise_median(values):
    """Median over the first axis; even count -> mean of the two middle values (R14)."""
    a = np.sort(np.asarray(values, float), axis=0)
    k = a.shape[0]
    if k % 2 == 1:
        return a[k // 2]
    return 0.5 * (a[k // 2 - 1] + a[k // 2])


def kl_deviation(a, A, b, B) -> float:
    """eq. KL: requires B invertible, A need not be."""
    p = A.shape[0]
    Bi = np.linalg.inv(B)
    M = A @ Bi
    sign, ld = np.linalg.slogdet(M)
    d = np.asarray(a) - np.asarray(b)
    logdet = ld if sign > 0 else (np.nan if sign == 0 else np.nan)
    return float(np.trace(M) - p - logdet + d @ Bi @ d)


def kl_rank_key(mu_med, S_med, mu_l, S_l) -> float:
    """KL minus the terms common to every block: tr(S_med S_l^-1) + log det S_l + quad.

    Ranking-identical to eq. KL (reading R15) and defined when S_med is not PD.
    """
    Si = np.linalg.inv(S_l)
    d = mu_med - mu_l
    sign, ld = np.linalg.slogdet(S_l)
    return float(np.trace(S_med @ Si) + ld + d @ Si @ d)


def select_and_pool(mus, Sigmas, ms, block_ids=None):
    """Steps 5-7.  Returns (mu_raw, Sigma_raw, kept block ids, keys)."""
    q = len(mus)
    if block_ids is None:
        block_ids = list(range(q))
    mus = [np.asarray(x, float) for x in mus]
    Sigmas = [np.asarray(x, float) for x in Sigmas]
    mu_med = entrywise_median(mus)
    S_med = entrywise_median(Sigmas)
    keys = [kl_rank_key(mu_med, S_med, mus[l], Sigmas[l]) for l in range(q)]
    order = sorted(range(q), key=lambda l: (keys[l], block_ids[l]))
    keep = sorted(order[: int(math.ceil(q / 2))], key=lambda l: block_ids[l])
    # single-pass pooling (eqs. covpool), folded in block-id order
    l0 = keep[0]
    Lam = (ms[l0] - 1) * Sigmas[l0]
    mu_p = mus[l0].copy()
    n_p = ms[l0]
    for l in keep[1:]:
        m = ms[l]
        dmu = mus[l] - mu_p
        Lam = Lam + (m - 1) * Sigmas[l] + np.outer(dmu, dmu) * (n_p * m / (n_p + m))
        mu_p = (n_p * mu_p + m * mus[l]) / (n_p + m)
        n_p = n_p + m
    return mu_p, Lam / (n_p - 1), [block_ids[l] for l in keep], keys
