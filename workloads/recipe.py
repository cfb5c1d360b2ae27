"""Seeded synthetic inputs -- the one module both the oracle side and the CUDA side draw from.

This module holds NO arithmetic of the paper's method (no partitioning, no SpMV/SpAdd/SpMM);
it only manufactures sorted CSR / DCSR operands and dense vectors.  Every random number is a
counter-based hash of (seed, stream, a, b), so a row or an entry can be regenerated on its own
and the CUDA generator (workloads/gen.cu) reproduces these arrays bit for bit.

Recipe (SURVEY.md 8(d) with reading R14):
  * row degrees: rank-Zipf with exponent s = 1, deg(r) = clamp(cdiv // (pi(r)+1), min_deg, cap)
    where pi is a seeded Feistel bijection on [0, M) (heavy rows scattered) and cdiv is found by
    bisection so that sum(deg) ~= target ("power-law matrices ... lower exponents indicate higher
    skew", P:2227 -- a degree-distribution exponent gamma = 1 + 1/s = 2);
  * columns: stratified sampling inside a window of width W >= deg -- one column per stratum,
    hence strictly increasing and distinct by construction:
      local   W = min(N, max(4 deg, 4096)) centred on the scaled diagonal r*N/M (SuiteSparse-like)
      uniform W = N (x-gather stress)
      web     half the rows: first deg//2 entries in the popular column block [0, N/64), the rest
              over [N/64, N); the other rows local (web-graph-shaped hubs)
  * values: 0.5 + u * 2^-24 with 24 random bits (exact in fp32 and fp64), or small integers.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
K_SEED = 0x9E3779B97F4A7C15
K_STREAM = 0xD1B54A32D192ED03
K_A = 0xABC98388FB8FAC03
K_B = 0x8CB92BA72F3D8DD7

# stream ids (must match gen.cu)
S_PERM, S_COL, S_VAL, S_X, S_B, S_KIND, S_OUTER, S_REUSE_B, S_REUSE_C, S_PICK_C = range(1, 11)


def _u64(x):
    return np.asarray(x).astype(np.uint64, copy=False)


def mix64(z):
    """splitmix64 finalizer on uint64 arrays (wrap-around arithmetic)."""
    z = _u64(z).copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def hash4(seed, stream, a, b):
    """Counter-based hash of (seed, stream, a, b) -> uint64 array."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed & M64) * np.uint64(K_SEED)
             + np.uint64(stream) * np.uint64(K_STREAM)
             + _u64(a) * np.uint64(K_A)
             + _u64(b) * np.uint64(K_B))
    return mix64(z)


# ------------------------------------------------------------------ permutation
def _feistel_bits(n):
    b = max(2, int(n - 1).bit_length())
    return (b + 1) // 2


def feistel_perm(x, n, seed):
    """Seeded bijection on [0, n): 4-round balanced Feistel on 2h bits with cycle walking."""
    x = _u64(x).copy()
    if n <= 1:
        return np.zeros_like(x)
    h = _feistel_bits(n)
    mask = np.uint64((1 << h) - 1)
    hh = np.uint64(h)
    todo = np.ones(x.shape, dtype=bool)
    while True:
        y = x[todo]
        for rnd in range(4):
            L = y >> hh
            R = y & mask
            F = hash4(seed, S_PERM, R, rnd) & mask
            y = (R << hh) | (L ^ F)
        x[todo] = y
        todo = x >= np.uint64(n)
        if not todo.any():
            return x


# ------------------------------------------------------------------ degrees
def sum_floor_div(cdiv, m, cap, min_deg=0):
    """sum_{q=0}^{m-1} clamp(cdiv // (q+1), min_deg, cap), O(sqrt(cdiv)) block summation."""
    total = 0
    d = 1
    lim = min(m, cdiv)
    while d <= lim:
        v = cdiv // d
        dmax = min(cdiv // v, lim)
        total += max(min(v, cap), min_deg) * (dmax - d + 1)
        d = dmax + 1
    if m > lim:
        total += max(0, min_deg) * (m - lim)
    return total


def find_cdiv(m, target, cap, min_deg=0):
    lo, hi = 0, 1
    while sum_floor_div(hi, m, cap, min_deg) < target and hi < (1 << 62):
        hi *= 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if sum_floor_div(mid, m, cap, min_deg) < target:
            lo = mid
        else:
            hi = mid
    return hi


def degrees(m, cdiv, cap, seed, min_deg=0):
    r = np.arange(m, dtype=np.uint64)
    rank = feistel_perm(r, m, seed).astype(np.int64)
    d = cdiv // (rank + 1)
    return np.clip(d, min_deg, cap).astype(np.int64)


def pos_from_degrees(deg):
    pos = np.zeros(len(deg) + 1, dtype=np.int64)
    np.cumsum(deg, out=pos[1:])
    return pos


# ------------------------------------------------------------------ columns
def _strata(w0, w, d, k):
    lo = w0 + (k * w) // d
    hi = w0 + ((k + 1) * w) // d
    return lo, hi


def _pick(seed, stream, r, k, lo, hi):
    h = hash4(seed, stream, r, k)
    return lo + (h % _u64(hi - lo)).astype(np.int64)


def entry_rows(pos):
    deg = np.diff(pos)
    return np.repeat(np.arange(len(deg), dtype=np.int64), deg)


def columns(kind, m, n, seed, pos, stream=S_COL, rows=None):
    """Column coordinates for every entry of a CSR pattern with row pointer `pos` (int32)."""
    if rows is None:
        rows = entry_rows(pos)
    k = np.arange(pos[-1], dtype=np.int64) - pos[rows]
    d = (pos[rows + 1] - pos[rows]).astype(np.int64)
    r = rows.astype(np.int64)
    if kind == "uniform":
        w = np.full_like(d, n)
        w0 = np.zeros_like(d)
    else:
        w = np.minimum(n, np.maximum(4 * d, 4096))
        centre = (r * n) // m
        w0 = np.clip(centre - w // 2, 0, n - w)
    lo, hi = _strata(w0, w, d, k)
    col = _pick(seed, stream, r, k, lo, hi)
    if kind == "web":
        npop = max(1, n // 64)
        d1 = d // 2
        web = ((hash4(seed, S_KIND, r, 0) & np.uint64(1)) == np.uint64(1)) & (d1 <= npop) & (d - d1 <= n - npop) & (d1 > 0)
        first = k < d1
        lo1, hi1 = _strata(np.zeros_like(d), np.full_like(d, npop), np.maximum(d1, 1), k)
        lo2, hi2 = _strata(np.full_like(d, npop), np.full_like(d, n - npop), np.maximum(d - d1, 1), k - d1)
        lo_w = np.where(first, lo1, lo2)
        hi_w = np.where(first, hi1, hi2)
        col_w = _pick(seed, stream, r, k, lo_w, np.maximum(hi_w, lo_w + 1))
        col = np.where(web, col_w, col)
    dense = d >= n
    col = np.where(dense, k, col)
    return col.astype(np.int32)


def values(seed, stream, idx, dtype, mode="uniform", kmax=4):
    h = hash4(seed, stream, idx, 0)
    bits = (h >> np.uint64(40)).astype(np.int64)              # 24 random bits
    if mode == "uniform":
        v = 0.5 + bits.astype(np.float64) * (2.0 ** -24)
    else:
        mag = 1 + bits % kmax
        sign = np.where((h >> np.uint64(63)) == np.uint64(1), -1, 1)
        v = (mag * sign).astype(np.float64)
    return v.astype(dtype)


def outer_rows(m, nouter, seed):
    """nouter distinct sorted stored-row coordinates in [0, m): one per stratum of width m/nouter."""
    k = np.arange(nouter, dtype=np.int64)
    lo = (k * m) // nouter
    hi = ((k + 1) * m) // nouter
    return _pick(seed, S_OUTER, k, 0, lo, hi).astype(np.int32)
