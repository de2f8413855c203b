"""ORACLE (test infrastructure only) -- the replayable index stream, written from
the text specification in include/ils.h ("Index stream"), independently of the
CUDA path (no shared code, tables or constants generators).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg
may import this module.

The paper draws its indices with MATLAB's rand (Alg. 2 steps
8/10; Alg. 5 steps 7-8). To let an oracle replay the GPU's
exact index sequence both sides implement the same counter-based generator
(Philox4x32-10, Salmon et al. SC'11) and the same integer sampler:

* column-norm probability ||A1_(j)||^2/||A1||_F^2 (PAPER.md:199-202, :227-230,
  Eq. Sec3.21.1) -> integer weights W_j = max(1, floor(N_j/N_max * 2^32)) with
  N_j summed sequentially (reading R7);
* alpha_t uniform on [n] (reading R8);
* the "uniformly random" size-alpha subset -> prefix of a keyed
  8-round Feistel permutation of [n] with cycle walking (reading R9).
"""
from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85

TAG_RKRGS = 1
TAG_SCD_A = 2
TAG_SCD_B = 3
TAG_SCD_C = 4
TAG_RCD = 6
TAG_SUBSET = 7
SUBSET_EXACT = 0x10
FEISTEL_ROUNDS = 8


def philox4x32_10(ctr, key):
    """Philox4x32 with 10 rounds. ctr: (..., 4) uint32-valued array, key: (k0, k1).

    Round: (c0,c1,c2,c3) -> (hi(M1*c2)^c1^k0, lo(M1*c2), hi(M0*c0)^c3^k1, lo(M0*c0)),
    key bumped by (W0, W1) between rounds.
    """
    c = np.array(ctr, dtype=np.uint64) & np.uint64(M32)
    c0, c1, c2, c3 = (c[..., i].copy() for i in range(4))
    k0 = int(key[0]) & M32
    k1 = int(key[1]) & M32
    for r in range(10):
        p0 = np.uint64(PHILOX_M0) * c0
        p1 = np.uint64(PHILOX_M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(M32)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(M32)
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0)
        k0 = (k0 + PHILOX_W0) & M32
        k1 = (k1 + PHILOX_W1) & M32
    return np.stack([c0, c1, c2, c3], axis=-1)


def draw(seed: int, k: int, t, tag: int):
    """Philox output words for counter (t_lo, t_hi, k, tag), key (seed_lo, seed_hi).
    t may be an int or an integer array. Returns uint64 array (..., 4) of 32-bit words."""
    t = np.asarray(t, dtype=np.uint64)
    ctr = np.stack([t & np.uint64(M32), t >> np.uint64(32),
                    np.full_like(t, k & M32), np.full_like(t, tag)], axis=-1)
    return philox4x32_10(ctr, (seed & M32, (seed >> 32) & M32))


def column_norms_sq(A1: np.ndarray) -> np.ndarray:
    """N_j = sum_i A1[i,j]^2, summed sequentially over i = 0..p-1, each square
    rounded before the add (no fused multiply-add): the definition of
    ||A1_(j)||_2^2 in a fixed summation order, so that both sides agree bit for bit."""
    N = np.zeros(A1.shape[1])
    for i in range(A1.shape[0]):      # sequential over rows i = 0..p-1
        N = N + A1[i] * A1[i]
    return N


def column_norms_sq_csc(indptr: np.ndarray, data: np.ndarray, n: int) -> np.ndarray:
    """The same N_j for A1 stored by columns (CSC with ascending row indices per column, e.g.
    configs[3]): the stored entries of column j are added in ascending row order, each square
    rounded before the add. The structural zeros the dense loop also adds leave every partial sum
    unchanged (s + 0.0 = s exactly), so this equals column_norms_sq on the densified matrix bit for
    bit (pinned in tests/test_oracle_pins.py). Rank r of every column is added in pass r."""
    indptr = np.asarray(indptr, dtype=np.int64)
    cnt = np.diff(indptr)
    N = np.zeros(n)
    for r in range(int(cnt.max()) if n else 0):
        cols = np.flatnonzero(cnt > r)
        v = data[indptr[cols] + r]
        N[cols] = N[cols] + v * v
    return N


def weights_prefix(N: np.ndarray):
    """Integer weights W_j = max(1, floor(N_j / N_max * 2^32)) and inclusive prefix sums
    S_j = sum_{i<=j} W_i (Python ints, exact)."""
    if np.any(N <= 0):
        raise ValueError("zero column in A1 (||A1_(j)||^2 = 0)")
    nmax = float(np.max(N))
    W = [max(1, int(np.floor(np.ldexp(float(v) / nmax, 32)))) for v in N]
    S, acc = [], 0
    for w in W:
        acc += w
        S.append(acc)
    return W, S


def sample_weighted(U: int, S) -> int:
    """j = min{ j : S_j > v }, v = floor(U * S_total / 2^64) (U a 64-bit uniform).
    P(j) = W_j / S_total up to 2^-64 relative bias."""
    v = (int(U) * int(S[-1])) >> 64
    lo, hi = 0, len(S) - 1
    while lo < hi:                     # smallest j with S[j] > v
        mid = (lo + hi) // 2
        if S[mid] > v:
            hi = mid
        else:
            lo = mid + 1
    return lo


def rk_rgs_indices(seed: int, k: int, t0: int, count: int, S):
    """(j1, j2) for inner steps t0..t0+count-1 of outer iteration k (Alg. 2 steps 8, 10):
    U1 = x1<<32 | x0 -> j1 ; U2 = x3<<32 | x2 -> j2 (independent draws, reading R6)."""
    X = draw(seed, k, np.arange(t0, t0 + count, dtype=np.uint64), TAG_RKRGS)
    j1 = [sample_weighted((int(x[1]) << 32) | int(x[0]), S) for x in X]
    j2 = [sample_weighted((int(x[3]) << 32) | int(x[2]), S) for x in X]
    return np.array(j1, dtype=np.int64), np.array(j2, dtype=np.int64)


def rcd_indices(seed: int, k: int, t0: int, count: int, S):
    """Weighted single index for SP-RCD (alpha = 1 with column-norm probabilities,
    PAPER.md:460-475 and Remark 4.1 PAPER.md:506-510)."""
    X = draw(seed, k, np.arange(t0, t0 + count, dtype=np.uint64), TAG_RCD)
    return np.array([sample_weighted((int(x[1]) << 32) | int(x[0]), S) for x in X],
                    dtype=np.int64)


def _mix32(x):
    """mix32(x) on uint64 arrays holding 32-bit values (all arithmetic mod 2^32)."""
    m = np.uint64(M32)
    x = (x * np.uint64(0x85EBCA6B)) & m
    x ^= x >> np.uint64(13)
    x = (x * np.uint64(0xC2B2AE35)) & m
    x ^= x >> np.uint64(16)
    return x


def feistel_params(n: int):
    b = 0
    while (1 << b) < n:
        b += 1
    h = (b + 1) // 2
    return h, (1 << h) - 1


def feistel_forward(i, keys, n: int):
    """pi(i) for an int or integer array i: 8-round balanced Feistel on 2h bits
    (h = ceil(ceil(log2 n)/2)), round (L, R) -> (R, L ^ F(R, K_r)),
    F(R, K) = mix32(R ^ K) & (2^h - 1), cycle-walked until the value lies in [0, n)."""
    x = np.array(i, dtype=np.uint64)
    if n == 1:
        return np.zeros_like(x)
    h, mask = feistel_params(n)
    H, MASK = np.uint64(h), np.uint64(mask)

    def E(v):
        L, R = v >> H, v & MASK
        for r in range(FEISTEL_ROUNDS):
            L, R = R, L ^ (_mix32(R ^ np.uint64(int(keys[r]))) & MASK)
        return (L << H) | R

    x = E(x)
    out = np.atleast_1d(x)
    while True:                       # cycle walking: re-encrypt values outside [0, n)
        bad = out >= np.uint64(n)
        if not bad.any():
            break
        out[bad] = E(out[bad])
    return out.reshape(np.shape(x))


def scd_alpha_keys(seed: int, k: int, t: int, n: int, alpha_mode: int = 0, alpha_fixed: int = 1):
    """alpha_t and the eight Feistel round keys for SCD step t of outer iteration k
    (Alg. 5 steps 7-8). alpha_mode 0: uniform on {1..n} (alpha = 1 + hi32(x0 * n) of the
    tag-A draw); 1: fixed min(alpha_fixed, n). Round keys K0..K7 = A.x1..x3, B.x0..x3, C.x0."""
    xa = draw(seed, k, t, TAG_SCD_A)
    xb = draw(seed, k, t, TAG_SCD_B)
    xc = draw(seed, k, t, TAG_SCD_C)
    if alpha_mode == 0:
        alpha = 1 + ((int(xa[0]) * n) >> 32)
    else:
        alpha = min(int(alpha_fixed), n)
    keys = [int(v) for v in (xa[1], xa[2], xa[3], xb[0], xb[1], xb[2], xb[3], xc[0])]
    return alpha, keys


def subset_keys(seed: int, k: int, t: int, n: int):
    """Exact-subset keys (include/ils.h ILS_SUBSET_EXACT): u_s = word (s mod 4) of the Philox draw
    with counter (t_lo, t_hi, k, 7 + 256 * floor(s / 4)), key (seed_lo, seed_hi)."""
    nb = (n + 3) // 4
    b = np.arange(nb, dtype=np.uint64)
    t = int(t)
    ctr = np.stack([np.full(nb, t & M32, dtype=np.uint64), np.full(nb, (t >> 32) & M32, dtype=np.uint64),
                    np.full(nb, k & M32, dtype=np.uint64), np.uint64(TAG_SUBSET) + np.uint64(256) * b], axis=-1)
    X = philox4x32_10(ctr, (seed & M32, (seed >> 32) & M32))
    return X.reshape(-1)[:n]


def scd_subset(seed: int, k: int, t: int, n: int, alpha_mode: int = 0, alpha_fixed: int = 1):
    """tau_t = { pi(0), ..., pi(alpha_t - 1) } (Alg. 5 step 8). alpha_mode | SUBSET_EXACT: the
    alpha_t coordinates with the smallest (key, index) -- an exactly uniform size-alpha_t subset
    (Alg. 5 step 8 read literally), for the study of reading R9."""
    if alpha_mode & SUBSET_EXACT:
        alpha, _ = scd_alpha_keys(seed, k, t, n, alpha_mode & 0xF, alpha_fixed)
        u = subset_keys(seed, k, t, n)
        order = np.lexsort((np.arange(n), u))      # by key, then by index
        return alpha, np.sort(order[:alpha].astype(np.int64))
    alpha, keys = scd_alpha_keys(seed, k, t, n, alpha_mode, alpha_fixed)
    tau = feistel_forward(np.arange(alpha, dtype=np.uint64), keys, n)
    return alpha, np.sort(tau.astype(np.int64))
