"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws random
numbers (numpy PCG64 ``default_rng``) in the shapes and distributions of the
workloads named in BASELINE.json ``configs`` (SURVEY.md §8(d) "Generators").
Both the CUDA path and the CPU oracle consume the same bytes produced here;
neither side generates its own inputs.

Recipes (DESIGN.md §"Input recipe"):

========  ======================================================================
cfg1      a, b = rng(1001).random(n, f32) in [0, 1)           vadd -> reduce
cfg2      keys = rng(1002).integers(0, 256, n, int32) uniform   histogram
          variants: all-zero keys, geometric(0.5)-1 clipped to 255 (skew)
cfg3      u = rng(1003).random(n, f32) in [0, 1)               Black-Scholes
          (APARAPI mapping u -> S, K, T, R, sigma lives in the kernel/oracle)
cfg4      A, B = rng(1004).random((M, K)), ((K, N)) f32 U[0,1)   SGEMM
          variants: U[-1, 1) (seed 1014), integers in [-8, 8] (seed 1024)
cfg5      positions uniform in the unit ball (rng(1005)), m = 1/N, v = 0
          packed float4 (x, y, z, m) / (vx, vy, vz, 0)           N-body
========  ======================================================================
"""
from __future__ import annotations

import numpy as np

SEED_VADD = 1001
SEED_HIST = 1002
SEED_BS = 1003
SEED_SGEMM = 1004
SEED_NBODY = 1005
SEED_SGEMM_SIGNED = 1014
SEED_SGEMM_INT = 1024

# BASELINE.json configs, full sizes
CFG1_N = 1 << 20
CFG2_N = 1 << 28
CFG2_BINS = 256
CFG3_N = 1 << 26
CFG4_MNK = 8192
CFG5_N = 1 << 17
CFG5_STEPS = 10
# N-body constants (SURVEY.md §8(c)-N proposal; reading R16)
NBODY_DT = 0.016
NBODY_EPS2 = 0.01
NBODY_G = 1.0


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def uniform_f32(n: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    r = rng(seed).random(n, dtype=np.float32)
    if lo != 0.0 or hi != 1.0:
        r = (r * np.float32(hi - lo) + np.float32(lo)).astype(np.float32)
    return r


def vadd_inputs(n: int = CFG1_N, seed: int = SEED_VADD):
    g = rng(seed)
    a = g.random(n, dtype=np.float32)
    b = g.random(n, dtype=np.float32)
    return a, b


def hist_keys(n: int = CFG2_N, nbins: int = CFG2_BINS, seed: int = SEED_HIST,
              dist: str = "uniform") -> np.ndarray:
    g = rng(seed)
    if dist == "uniform":
        return g.integers(0, nbins, n, dtype=np.int32)
    if dist == "zeros":
        return np.zeros(n, dtype=np.int32)
    if dist == "geometric":
        k = g.geometric(0.5, n) - 1
        return np.minimum(k, nbins - 1).astype(np.int32)
    if dist == "with_out_of_range":
        # keys in [-8, nbins + 8): the out-of-range ones must be ignored
        return g.integers(-8, nbins + 8, n, dtype=np.int32)
    raise ValueError(dist)


def bs_rand(n: int = CFG3_N, seed: int = SEED_BS) -> np.ndarray:
    return rng(seed).random(n, dtype=np.float32)


def sgemm_inputs(m: int, n: int, k: int, dist: str = "unit", seed: int | None = None):
    if dist == "unit":
        g = rng(SEED_SGEMM if seed is None else seed)
        a = g.random((m, k), dtype=np.float32)
        b = g.random((k, n), dtype=np.float32)
    elif dist == "signed":
        g = rng(SEED_SGEMM_SIGNED if seed is None else seed)
        a = (g.random((m, k), dtype=np.float32) * 2 - 1).astype(np.float32)
        b = (g.random((k, n), dtype=np.float32) * 2 - 1).astype(np.float32)
    elif dist == "int":
        g = rng(SEED_SGEMM_INT if seed is None else seed)
        a = g.integers(-8, 9, (m, k)).astype(np.float32)
        b = g.integers(-8, 9, (k, n)).astype(np.float32)
    else:
        raise ValueError(dist)
    return np.ascontiguousarray(a), np.ascontiguousarray(b)


def nbody_state(n: int = CFG5_N, seed: int = SEED_NBODY):
    """float4 positions (x, y, z, m) uniform in the unit ball, m = 1/n; v = 0."""
    g = rng(seed)
    d = g.standard_normal((n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = g.random(n) ** (1.0 / 3.0)
    pos = np.empty((n, 4), dtype=np.float32)
    pos[:, :3] = (d * r[:, None]).astype(np.float32)
    pos[:, 3] = np.float32(1.0 / n)
    vel = np.zeros((n, 4), dtype=np.float32)
    return pos, vel


def shard_range(n: int, rank: int, world: int):
    """Index range [lo, hi) of rank's shard: contiguous, sizes differ by <= 1.

    This is the partitioning of SURVEY.md §8(e) ("index range
    [r*N/P, (r+1)*N/P)"); it is pure bookkeeping, no method arithmetic.
    """
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


# ----------------------------------------------------------- NEXT rows (§8(f))
CORR_TERMS = 1024          # P:494 "1024 Terms and 16384 Documents"
CORR_DOCS = 16384
SPMV_N = 44609             # P:487 bcsstk32: 44609 x 44609, 1029655 non-zeros
SPMV_NNZ = 1029655
CONV_N = 2048              # P:489 "2048 x 2048 image with a 5 x 5 filter"


def corr_bitsets(terms: int = CORR_TERMS, docs: int = CORR_DOCS, density: float = 0.5, seed: int = 1006):
    """(terms, docs/32) uint32: bit d%32 of word d/32 = document d contains the term."""
    assert docs % 32 == 0
    bits = rng(seed).random((terms, docs)) < density
    packed = np.packbits(bits.reshape(terms, docs // 8, 8), axis=-1, bitorder="little")
    return np.ascontiguousarray(packed.reshape(terms, docs // 8)).view(np.uint32).reshape(terms, docs // 32)


def banded_csr(n: int = SPMV_N, nnz: int = SPMV_NNZ, bandwidth: int = 1600, seed: int = 1007):
    """Synthetic stand-in for bcsstk32 (no dataset offline): n x n, ~nnz
    non-zeros, symmetric pattern inside a band, every diagonal present,
    values U[-1, 1).  Returns (row_ptr int32[n+1], col int32[nnz'], val f32[nnz'])."""
    g = rng(seed)
    per_row = max(0, (nnz - n) // (2 * n))          # off-diagonal pairs per row
    i = np.repeat(np.arange(n), per_row)
    j = i + g.integers(1, bandwidth, i.size)
    keep = j < n
    i, j = i[keep], j[keep]
    rows = np.concatenate([np.arange(n), i, j])
    cols = np.concatenate([np.arange(n), j, i])
    key = np.unique(rows.astype(np.int64) * n + cols)
    rows, cols = (key // n).astype(np.int32), (key % n).astype(np.int32)
    row_ptr = np.zeros(n + 1, np.int32)
    np.add.at(row_ptr, rows + 1, 1)
    row_ptr = np.cumsum(row_ptr, dtype=np.int64).astype(np.int32)
    val = (g.random(cols.size, dtype=np.float32) * 2 - 1).astype(np.float32)
    return row_ptr, cols, val


def powerlaw_csr(n: int, mean_nnz: float = 8.0, seed: int = 1017, alpha: float = 1.6,
                 empty_frac: float = 0.1, long_rows=(), ncols: int | None = None):
    """Irregular CSR input: row lengths from a discrete power law (Pareto
    tail with exponent `alpha`, scaled to about `mean_nnz` per row, capped
    at ncols), a fraction `empty_frac` of rows empty, and explicit long rows
    `long_rows = ((row, length), ...)`; columns uniform in [0, ncols), sorted
    and unique within a row; values U[-1, 1).  (The irregular row-length mix
    of a real sparse matrix such as bcsstk32, which is unavailable offline.)
    Returns (row_ptr int32[n+1], col int32[nnz], val f32[nnz])."""
    ncols = n if ncols is None else ncols
    g = rng(seed)
    lens = np.floor(g.pareto(alpha, n) * mean_nnz * (alpha - 1) / alpha * 1.5).astype(np.int64)
    lens = np.minimum(lens, ncols)
    lens[g.random(n) < empty_frac] = 0
    for r, ln in long_rows:
        lens[r] = min(ln, ncols)
    cols = []
    for r in np.nonzero(lens)[0]:
        ln = int(lens[r])
        if ln * 4 >= ncols:
            c = np.sort(g.choice(ncols, ln, replace=False))
        else:
            c = np.unique(g.integers(0, ncols, ln + ln // 8 + 4))[:ln]
            lens[r] = c.size
        cols.append(c)
    row_ptr = np.zeros(n + 1, np.int64)
    row_ptr[1:] = np.cumsum(lens)
    col = (np.concatenate(cols) if cols else np.zeros(0, np.int64)).astype(np.int32)
    val = (g.random(col.size, dtype=np.float32) * 2 - 1).astype(np.float32)
    return row_ptr.astype(np.int32), col, val
