"""CPU ORACLE for the Jacc hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_1508_06791_b200`` + ``libjacc.so``) never imports it and
shares no code with it; the only shared module is ``synth`` (seeded input
generators, no method arithmetic).

Contents
--------
* ``jacc_oracle.c`` -- plain fp64 C loops for every kernel on the hot path
  (vector add, reduction, histogram, Black-Scholes, SGEMM, N-body), each
  citing the PAPER.md passage it follows.  Built by :func:`build` with gcc.
* ``graph_model.py`` -- the task-graph semantics: dependency inference,
  the transfer-elision model (counted copies) and the serial executor.

Every function is pinned in ``tests/test_oracle_pins.py`` /
``tests/test_graph_model.py`` against closed forms, brute force,
invariants or library routines; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "jacc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_I64P = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (no fast-math, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.oracle_num_threads.restype = ctypes.c_int
            L.oracle_set_num_threads.argtypes = [ctypes.c_int]
            L.oracle_vadd_f32.argtypes = [_F32P, _F32P, _F32P, _i64]
            L.oracle_reduce_sum_f32.argtypes = [_F32P, _i64, _f64, ctypes.POINTER(_f64)]
            L.oracle_reduce_sum_f32.restype = _f64
            L.oracle_histogram_i32.argtypes = [_I32P, _i64, ctypes.c_int32, _I32P, ctypes.c_int]
            L.oracle_bs_phi.argtypes = [_f64]
            L.oracle_bs_phi.restype = _f64
            L.oracle_bs_price.argtypes = [_f64] * 5 + [ctypes.POINTER(_f64)] * 2
            L.oracle_bs_params.argtypes = [_f64] + [ctypes.POINTER(_f64)] * 5
            L.oracle_blackscholes_f32.argtypes = [_F32P, _i64, _F64P, _F64P]
            L.oracle_blackscholes_soa_f32.argtypes = [_F32P] * 5 + [_i64, _F64P, _F64P]
            L.oracle_sgemm_rows_f32.argtypes = [_F32P, _F32P, _F64P, _i64, _i64, _i64,
                                                _i64, _i64, _i64, ctypes.c_void_p, _i64]
            L.oracle_nbody_accel.argtypes = [_F64P, _i64, _I64P, _i64, _f64, _f64, _F64P]
            L.oracle_nbody_steps.argtypes = [_F64P, _F64P, _i64, ctypes.c_int, _f64, _f64,
                                             _f64, _F64P, _I64P]
            L.oracle_conv2d_f32.argtypes = [_F32P, _i64, _i64, _F32P, ctypes.c_int, _F64P, _F64P]
            _U32P = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
            L.oracle_corr_popc.argtypes = [_U32P, _i64, _U32P, _i64, _i64, _I32P]
            L.oracle_spmv_csr_f32.argtypes = [_I32P, _I32P, _F32P, _F32P, _i64, _F64P, _F64P]
            _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the parallel oracle loops (results do not depend on it)."""
    lib().oracle_set_num_threads(int(n))


def _c(x, dt):
    return np.ascontiguousarray(x, dtype=dt)


# ---------------------------------------------------------------- kernels
def vadd(a, b):
    """c = fl32(a + b)."""
    a = _c(a, np.float32); b = _c(b, np.float32)
    assert a.shape == b.shape
    c = np.empty_like(a)
    lib().oracle_vadd_f32(a, b, c, a.size)
    return c


def reduce_sum(x, init: float = 0.0):
    """(s, sum|x|): s = init + sum x in fp64."""
    x = _c(x, np.float32).ravel()
    a = _f64(0.0)
    s = lib().oracle_reduce_sum_f32(x, x.size, float(init), ctypes.byref(a))
    return float(s), float(a.value)


def histogram(keys, nbins: int = 256, init=None):
    """bins[k] (+)= #{i: keys[i] == k}; out-of-range keys ignored (R11)."""
    keys = _c(keys, np.int32).ravel()
    if init is None:
        bins = np.zeros(nbins, dtype=np.int32)
        acc = 0
    else:
        bins = _c(init, np.int32).copy()
        assert bins.size == nbins
        acc = 1
    lib().oracle_histogram_i32(keys, keys.size, nbins, bins, acc)
    return bins


def bs_phi(x: float) -> float:
    return float(lib().oracle_bs_phi(float(x)))


def bs_price(S, K, T, R, sigma):
    c = _f64(); p = _f64()
    lib().oracle_bs_price(float(S), float(K), float(T), float(R), float(sigma),
                          ctypes.byref(c), ctypes.byref(p))
    return c.value, p.value


def bs_params(u: float):
    out = [_f64() for _ in range(5)]
    lib().oracle_bs_params(float(u), *[ctypes.byref(o) for o in out])
    return tuple(o.value for o in out)


def blackscholes(rand):
    """(call, put) in fp64 for the APARAPI mapping of rand (R12)."""
    r = _c(rand, np.float32).ravel()
    call = np.empty(r.size, np.float64); put = np.empty(r.size, np.float64)
    lib().oracle_blackscholes_f32(r, r.size, call, put)
    return call, put


def blackscholes_soa(S, K, T, R, sigma):
    arrs = [_c(v, np.float32).ravel() for v in (S, K, T, R, sigma)]
    n = arrs[0].size
    call = np.empty(n, np.float64); put = np.empty(n, np.float64)
    lib().oracle_blackscholes_soa_f32(*arrs, n, call, put)
    return call, put


def sgemm_rows(A, B, rows=None):
    """fp64 C[rows, :] = A[rows, :] . B (R13)."""
    A = _c(A, np.float32); B = _c(B, np.float32)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    if rows is None:
        C = np.empty((M, N), np.float64)
        lib().oracle_sgemm_rows_f32(A, B, C, M, N, K, K, N, N, None, 0)
    else:
        r = _c(rows, np.int64).ravel()
        C = np.empty((r.size, N), np.float64)
        lib().oracle_sgemm_rows_f32(A, B, C, M, N, K, K, N, N,
                                    r.ctypes.data_as(ctypes.c_void_p), r.size)
    return C


def nbody_accel(pos, targets=None, eps2: float = 0.01, G: float = 1.0):
    """fp64 accelerations of `targets` due to all bodies in pos (n x 4)."""
    p = _c(pos, np.float64).reshape(-1, 4)
    n = p.shape[0]
    t = np.arange(n, dtype=np.int64) if targets is None else _c(targets, np.int64).ravel()
    acc = np.empty((t.size, 3), np.float64)
    lib().oracle_nbody_accel(p, n, t, t.size, eps2, G, acc)
    return acc


def nbody_steps(pos, vel, steps: int, dt: float = 0.016, eps2: float = 0.01, G: float = 1.0):
    """fp64 symplectic Euler from the (fp32) initial state; returns (pos, vel)."""
    p = _c(pos, np.float64).reshape(-1, 4).copy()
    v = _c(vel, np.float64).reshape(-1, 4).copy()
    n = p.shape[0]
    scratch = np.empty((n, 3), np.float64)
    tgt = np.arange(n, dtype=np.int64)
    lib().oracle_nbody_steps(p, v, n, int(steps), dt, eps2, G, scratch, tgt)
    return p, v


def conv2d(img, filt):
    """fp64 (out, sum|f||img|): zero-padded true 2D convolution, same size
    (reading R20)."""
    img = _c(img, np.float32)
    filt = _c(filt, np.float32)
    H, W = img.shape
    k = filt.shape[0]
    assert filt.shape == (k, k) and k % 2 == 1
    out = np.empty((H, W), np.float64)
    ab = np.empty((H, W), np.float64)
    lib().oracle_conv2d_f32(img, H, W, filt, k // 2, out, ab)
    return out, ab


def halo_band(img, lo: int, hi: int, r: int):
    """The row band [lo, hi) of img with its r halo rows above and below,
    zeros past the image -- what JACC_OP_HALO_EXCHANGE_F32 assembles on the
    rank owning that band (include/jacc.h; SURVEY §8(f) f1 "shards by row
    bands with a 2-row halo exchange").  Plain slicing, no arithmetic."""
    img = _c(img, np.float32)
    H, W = img.shape
    ext = np.zeros((hi - lo + 2 * r, W), np.float32)
    for y in range(lo - r, hi + r):
        if 0 <= y < H:
            ext[y - (lo - r)] = img[y]
    return ext


def corr_popc(A, B=None):
    """C[i][j] = sum_w popcount(A[i][w] & B[j][w]) (R21).
    A: (ta, words) uint32 bitsets; B defaults to A."""
    A = _c(A, np.uint32)
    B = A if B is None else _c(B, np.uint32)
    assert A.shape[1] == B.shape[1]
    C = np.empty((A.shape[0], B.shape[0]), np.int32)
    lib().oracle_corr_popc(A, A.shape[0], B, B.shape[0], A.shape[1], C)
    return C


def spmv_csr(row_ptr, col, val, x):
    """fp64 (y, sum|a x|) with y = A x, A in CSR (R22)."""
    rp = _c(row_ptr, np.int32); cl = _c(col, np.int32)
    v = _c(val, np.float32); xx = _c(x, np.float32)
    n = rp.size - 1
    y = np.empty(n, np.float64); ab = np.empty(n, np.float64)
    lib().oracle_spmv_csr_f32(rp, cl, v, xx, n, y, ab)
    return y, ab
