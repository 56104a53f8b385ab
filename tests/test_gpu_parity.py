"""GPU parity: the CUDA path (through the C-ABI, libjacc.so) vs the CPU oracle
on the same seeded inputs (synth/), element by element.

Tolerances (written here, derived in DESIGN.md §Tolerances from the
north_star: "bit-exact for integer histograms and indexing, and for floating
point within max relative error 1e-5 for maps and 1e-4 against an
fp64-accumulated oracle for reductions, SGEMM and N-body"):
  vadd       bit-exact (one IEEE fp32 add; stricter than the 1e-5 bar)
  reduce     |s - o| <= 1e-4 * sum|x|    (== relative error for x >= 0)
  histogram  bit-exact
  BS         |g - o| <= 1e-5 * (S + K e^{-RT})  per option (R12)
  SGEMM      U[0,1): max elementwise rel <= 1e-4; U[-1,1): normwise <= 1e-4
             and componentwise |C-R| <= 1e-4 (|A||B|); integer inputs exact
  N-body     after the steps: |dx_i| <= 1e-4 R (R = 1, ball radius),
             |dv_i| <= 1e-4 mean|v|; one step at full N: |da|/|a| <= 1e-4
"""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
J = pytest.importorskip("paper_1508_06791_b200")
from paper_1508_06791_b200 import jacc  # noqa: E402
from paper_1508_06791_b200.torch_glue import make_graph  # noqa: E402

R, W, RW = J.JACC_READ, J.JACC_WRITE, J.JACC_READWRITE


def _graph(**kw):
    g, _ = make_graph(0, **kw)
    return g


def _dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


# ------------------------------------------------------------------ vadd
@pytest.mark.parametrize("n", [1, 3, 31, 4097, 65539, 1 << 20])
def test_vadd_bit_exact(n):
    a, b = synth.vadd_inputs(n, seed=synth.SEED_VADD + n)
    c = np.zeros(n, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
    g.run()
    assert np.array_equal(c.view(np.uint32), oracle.vadd(a, b).view(np.uint32))
    g.destroy()


def test_vadd_ieee_specials_bit_exact():
    """One IEEE RN fp32 add per element, specials included (the oracle is
    pinned on them, tests/test_oracle_pins.py): +-Inf, NaN, -0, denormals
    (no flush to zero), overflow to Inf, Inf - Inf = NaN, max-normal sums."""
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 1.17549435e-38,
                   5.877472e-39, 3.4028235e38, -3.4028235e38, 1.0, -1.0, 2.0 ** -149 * 3,
                   2.0 ** 24, 0.5], np.float32)
    a = np.repeat(sp, sp.size)
    b = np.tile(sp, sp.size)
    # every pair, then a ragged tail that exercises the vector body and the
    # scalar remainder with specials in every lane position
    n = a.size * 257 + 3
    a = np.resize(a, n); b = np.resize(np.roll(b, 5), n)
    c = np.zeros(n, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
    g.run()
    g.destroy()
    ref = oracle.vadd(a, b)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(c), nan)
    assert np.array_equal(c[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    assert np.any(c.view(np.uint32) == np.float32(-0.0).view(np.uint32))       # -0 + -0 = -0
    assert np.any((c != 0) & (np.abs(c) < 1.17549435e-38))                      # denormal results kept


@pytest.mark.parametrize("off", [0, 4])
def test_vadd_256bit_path_bit_exact(off):
    """n >= 2^26: 32-byte aligned operands take the 256-bit kernel (off 0),
    16-byte aligned views the 128-bit one (off 4); random values with IEEE
    specials sprinkled in and a ragged tail of 13 -- bit-exact either way."""
    n = (1 << 26) + 13
    a, b = synth.vadd_inputs(n, seed=91)
    sp = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, 3.4028235e38, -3.4028235e38], np.float32)
    idx = synth.rng(92).integers(0, n, 4096)
    a[idx] = np.resize(sp, idx.size); b[idx[::-1]] = np.resize(sp, idx.size)
    a[-13:] = sp[:8].tolist() + [1.0] * 5
    da = torch.zeros(n + off, device="cuda"); db = torch.zeros(n + off, device="cuda")
    dc = torch.zeros(n + off, device="cuda")
    da[off:].copy_(torch.from_numpy(a)); db[off:].copy_(torch.from_numpy(b))
    g = _graph()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(da[off:], R), g.a(db[off:], R), g.a(dc[off:], W)])
    g.run()
    g.destroy()
    c = dc[off:].cpu().numpy()
    ref = oracle.vadd(a, b)
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(c), nan)
    assert np.array_equal(c[~nan].view(np.uint32), ref[~nan].view(np.uint32))
    assert float(dc[:off].abs().sum()) == 0


@pytest.mark.parametrize("off", [1, 2, 3])
def test_vadd_unaligned_device_args(off):
    n = 10007
    a, b = synth.vadd_inputs(n + off, seed=77)
    da, db = _dev(a), _dev(b)
    dc = torch.zeros(n + off, dtype=torch.float32, device="cuda")
    g = _graph()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(da[off:], R), g.a(db[off:], R), g.a(dc[off:], W)])
    g.run()
    assert np.array_equal(dc[off:].cpu().numpy(), oracle.vadd(a[off:], b[off:]))
    assert g.stats()["h2d_count"] == 0
    g.destroy()


@pytest.mark.parametrize("glob,group", [(32, 32), (1000, 64), (1 << 14, 128), (1 << 22, 1024), (0, 96)])
def test_schedule_invariance(glob, group):
    """R15 / P:162-165: the launch schedule (threads, group size) is advisory --
    fewer threads than iterations is a block-cyclic mapping -- and never
    changes a result: maps and the histogram are bitwise identical."""
    n = 300007
    a, b = synth.vadd_inputs(n, seed=5)
    keys = synth.hist_keys(n, seed=6)
    u = synth.bs_rand(n, seed=7)
    outs = []
    for sched in (None, jacc.jacc_schedule_t((glob, 0, 0), (group, 0, 0), 0)):
        c = np.zeros(n, np.float32); bins = np.zeros(256, np.int32)
        call = np.zeros(n, np.float32); put = np.zeros(n, np.float32)
        g = _graph()
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)], sched=sched)
        g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(bins, W)], jacc.jacc_hist_params_t(256), sched=sched)
        g.add_task(J.JACC_OP_BLACKSCHOLES_F32, [g.a(u, R), g.a(call, W), g.a(put, W)], sched=sched)
        g.run()
        g.destroy()
        outs.append((c, bins, call, put))
    for x, y in zip(outs[0], outs[1]):
        assert np.array_equal(x, y)


# ---------------------------------------------------------------- reduce
@pytest.mark.parametrize("n", [0, 1, 7, 4097, 1 << 20, (1 << 25) + 5])
def test_reduce_tolerance(n):
    x = synth.uniform_f32(n, 31 + n)
    s = np.zeros(1, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s, W)])
    g.run()
    ref, absum = oracle.reduce_sum(x)
    assert abs(float(s[0]) - ref) <= 1e-4 * absum + 1e-30
    g.destroy()


def test_reduce_pins_and_determinism():
    g = _graph()
    ones = np.ones(1 << 24, np.float32)     # all-ones, N <= 2^24: exact from any fp32 tree
    s = np.zeros(1, np.float32)
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(ones, R), g.a(s, W)])
    g.run()
    assert s[0] == float(1 << 24)
    g.destroy()
    x = np.arange(1, 1025, dtype=np.float32)   # S:287 -> 524800
    s = np.zeros(1, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s, W)])
    g.run()
    assert s[0] == 524800.0
    g.destroy()
    x = synth.uniform_f32(3 << 20, 5, -1, 1)
    outs = []
    for _ in range(3):
        s = np.zeros(1, np.float32)
        g = _graph()
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s, W)])
        g.run()
        outs.append(s[0])
        g.destroy()
    assert outs[0] == outs[1] == outs[2]


def test_reduce_readwrite_accumulates():
    x = synth.uniform_f32(100003, 9)
    s = np.array([1000.0], np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s, RW)])
    g.run()
    ref, absum = oracle.reduce_sum(x, init=1000.0)
    assert abs(float(s[0]) - ref) <= 1e-4 * (absum + 1000.0)
    assert g.stats()["memsets"] == 0
    g.destroy()


# ------------------------------------------------------------- histogram
@pytest.mark.parametrize("n,dist,nbins", [
    (0, "uniform", 256), (1, "uniform", 256), (255, "uniform", 256), (4099, "uniform", 256),
    ((1 << 20) + 3, "uniform", 256), (1 << 20, "zeros", 256), (1 << 20, "geometric", 256),
    ((1 << 20) + 1, "with_out_of_range", 256), (100000, "uniform", 100), (50000, "uniform", 1),
    (200001, "with_out_of_range", 1000), (100000, "uniform", 4096)])
def test_hist_bit_exact(n, dist, nbins):
    keys = synth.hist_keys(n, min(nbins, 256) if dist != "with_out_of_range" else nbins, seed=11 + n, dist=dist)
    if nbins == 4096:
        keys = synth.rng(3).integers(0, 4096, n, dtype=np.int32)
    bins = np.full(nbins, 7, np.int32)
    g = _graph()
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(bins, W)], jacc.jacc_hist_params_t(nbins))
    g.run()
    assert np.array_equal(bins, oracle.histogram(keys, nbins))
    g.destroy()


@pytest.mark.parametrize("mode", ["RW", "W"])
@pytest.mark.parametrize("off,n", [(1, 300007), (2, 300007), (3, 300007), (1, 3), (3, 6)])
def test_hist_unaligned_and_accumulate(off, n, mode):
    """Unaligned key views (head keys counted by the edge path into the
    workspace accumulator before the main kernel), W (bins assigned by the
    last block: no memset) and RW (host bins + counts), incl. views with
    fewer than 4 aligned keys."""
    keys = synth.hist_keys(n + off, 256, seed=4)
    dk = _dev(keys)
    init = np.arange(256, dtype=np.int32)
    bins = init.copy()
    g = _graph()
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(dk[off:], R), g.a(bins, RW if mode == "RW" else W)],
               jacc.jacc_hist_params_t(256))
    for _ in range(2):   # the accumulator must be re-zeroed by the first launch
        bins[:] = init
        g.run()
        want = oracle.histogram(keys[off:], 256, init=init if mode == "RW" else None)
        assert np.array_equal(bins, want)
    g.destroy()


@pytest.mark.parametrize("dist", ["zeros", "uniform", "with_out_of_range"])
def test_hist_counter_fold(dist):
    """The 16-bit lane counters' in-loop fold (before a counter can overflow):
    one block of 4 warps (advisory schedule) over 2^23 + 12345
    keys gives every warp > 2047 chunks of 32 keys per lane -- all keys in
    one bin loads a single counter to its limit before the fold."""
    n = (1 << 23) + 12345
    keys = synth.hist_keys(n, 256, seed=5, dist=dist)
    dk = _dev(keys)
    db = torch.zeros(256, dtype=torch.int32, device="cuda")
    g = _graph()
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(dk, R), g.a(db, W)], jacc.jacc_hist_params_t(256),
               sched=jacc.jacc_schedule_t((128, 0, 0), (128, 0, 0), 0))
    g.run()
    assert np.array_equal(db.cpu().numpy(), oracle.histogram(keys, 256))
    g.destroy()


def test_hist_full_size_config2():
    """BASELINE config 2 size (2^28 keys), the launch configuration bench.py times."""
    keys = synth.hist_keys()
    dk = _dev(keys)
    db = torch.zeros(256, dtype=torch.int32, device="cuda")
    g = _graph()
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(dk, R), g.a(db, W)], jacc.jacc_hist_params_t(256))
    g.run()
    assert np.array_equal(db.cpu().numpy(), oracle.histogram(keys, 256))
    assert int(db.sum()) == keys.size
    g.destroy()


# --------------------------------------------------------- Black-Scholes
def _bs_gate(call, put, oc, op, scale):
    assert np.all(np.abs(call - oc) <= 1e-5 * scale)
    assert np.all(np.abs(put - op) <= 1e-5 * scale)


@pytest.mark.parametrize("n", [1, 5, 4097, 1 << 20])
def test_bs_aparapi(n):
    u = synth.bs_rand(n, seed=synth.SEED_BS + n)
    call = np.zeros(n, np.float32); put = np.zeros(n, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_BLACKSCHOLES_F32, [g.a(u, R), g.a(call, W), g.a(put, W)])
    g.run()
    oc, op = oracle.blackscholes(u)
    S = 10 * u.astype(np.float64) + 100 * (1 - u.astype(np.float64))
    T = 1 * u.astype(np.float64) + 10 * (1 - u.astype(np.float64))
    Rr = 0.01 * u.astype(np.float64) + 0.05 * (1 - u.astype(np.float64))
    scale = S + S * np.exp(-Rr * T)
    _bs_gate(call, put, oc, op, scale)
    # put-call parity C - P = S - K e^{-RT} (exact in real arithmetic)
    assert np.all(np.abs((call - put) - (S - S * np.exp(-Rr * T))) <= 1e-5 * scale)
    g.destroy()


@pytest.mark.parametrize("off", [0, 4, 2, 1])
def test_bs_alignment_paths(off):
    """The three kernels of the APARAPI map: 256-bit I/O (32-byte aligned
    views), 128-bit (16-byte aligned), scalar (any) -- every one within the
    R12 gate of the oracle, tails included."""
    n = 20011
    u = synth.bs_rand(n, seed=77)
    base = torch.zeros(n + 8, device="cuda")
    du = base[off:off + n]
    du.copy_(torch.from_numpy(u))
    cbase = torch.zeros(n + 8, device="cuda"); pbase = torch.zeros(n + 8, device="cuda")
    dc, dp = cbase[off:off + n], pbase[off:off + n]
    g = _graph()
    g.add_task(J.JACC_OP_BLACKSCHOLES_F32, [g.a(du, R), g.a(dc, W), g.a(dp, W)])
    g.run()
    oc, op = oracle.blackscholes(u)
    uu = u.astype(np.float64)
    S = 10 * uu + 100 * (1 - uu); T = uu + 10 * (1 - uu); Rr = 0.01 * uu + 0.05 * (1 - uu)
    _bs_gate(dc.cpu().numpy(), dp.cpu().numpy(), oc, op, S + S * np.exp(-Rr * T))
    assert float(cbase[:off].abs().sum()) == 0 and float(cbase[off + n:].abs().sum()) == 0
    g.destroy()


def test_bs_full_size_config3_sampled():
    u = synth.bs_rand()
    du = _dev(u)
    dc = torch.empty_like(du); dp = torch.empty_like(du)
    g = _graph()
    g.add_task(J.JACC_OP_BLACKSCHOLES_F32, [g.a(du, R), g.a(dc, W), g.a(dp, W)])
    g.run()
    idx = synth.rng(9).integers(0, u.size, 1 << 16)
    idx = np.concatenate([idx, [0, 1, 2, 3, u.size - 1]])
    oc, op = oracle.blackscholes(u[idx])
    uu = u[idx].astype(np.float64)
    S = 10 * uu + 100 * (1 - uu); T = uu + 10 * (1 - uu); Rr = 0.01 * uu + 0.05 * (1 - uu)
    _bs_gate(dc.cpu().numpy()[idx], dp.cpu().numpy()[idx], oc, op, S + S * np.exp(-Rr * T))
    g.destroy()


def test_bs_soa_general_params():
    rng = np.random.default_rng(21)
    n = 20011
    S = rng.uniform(5, 200, n).astype(np.float32); K = rng.uniform(5, 200, n).astype(np.float32)
    T = rng.uniform(0.05, 10, n).astype(np.float32); Rr = rng.uniform(0, 0.1, n).astype(np.float32)
    V = rng.uniform(0.01, 0.9, n).astype(np.float32)
    call = np.zeros(n, np.float32); put = np.zeros(n, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_BLACKSCHOLES_SOA_F32, [g.a(S, R), g.a(K, R), g.a(T, R), g.a(Rr, R), g.a(V, R),
                                                 g.a(call, W), g.a(put, W)])
    g.run()
    oc, op = oracle.blackscholes_soa(S, K, T, Rr, V)
    scale = S.astype(np.float64) + K.astype(np.float64) * np.exp(-Rr.astype(np.float64) * T)
    _bs_gate(call, put, oc, op, scale)
    g.destroy()


# ------------------------------------------------------------------ SGEMM
def _sgemm(A, B, mode, device_args=False):
    M, K = A.shape
    N = B.shape[1]
    g = _graph()
    if device_args:
        dA, dB = _dev(A), _dev(B)
        dC = torch.empty((M, N), dtype=torch.float32, device="cuda")
        args = [g.a(dA, R), g.a(dB, R), g.a(dC, W)]
    else:
        C = np.zeros((M, N), np.float32)
        args = [g.a(A, R), g.a(B, R), g.a(C, W)]
    g.add_task(J.JACC_OP_SGEMM_F32, args, jacc.jacc_sgemm_params_t(M, N, K, K, N, N, mode, 0))
    g.run()
    out = dC.cpu().numpy() if device_args else C
    g.destroy()
    return out


# (1,1,1), (127,129,65): unaligned strides -> the pre-split path; the rest the
# CTA-pair path, incl. tiles mostly outside M / N and a K tail inside a block
SG_SHAPES = [(1, 1, 1), (127, 129, 65), (8, 16, 32), (200, 40, 20), (64, 300, 48), (256, 256, 256),
             (300, 520, 1000), (1024, 768, 2048)]


@pytest.mark.parametrize("mode", [J.JACC_SGEMM_FFMA, J.JACC_SGEMM_3XTF32], ids=["ffma", "3xtf32"])
def test_sgemm_strided_and_degenerate(mode):
    """Leading dimensions larger than the logical widths (sub-matrix views of
    padded storage, P:525 row-major with lda/ldb/ldc), and K = 0 (C = 0,
    beta = 0: every element written, none read)."""
    M, N, K, lda, ldb, ldc = 200, 300, 130, 136, 333, 301
    rng = synth.rng(91)
    Ast = rng.integers(-8, 9, (M, lda)).astype(np.float32)
    Bst = rng.integers(-8, 9, (K, ldb)).astype(np.float32)
    Cst = np.full((M, ldc), 7.0, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_SGEMM_F32, [g.a(Ast, R), g.a(Bst, R), g.a(Cst, W)],
               jacc.jacc_sgemm_params_t(M, N, K, lda, ldb, ldc, mode, 0))
    g.run(); g.destroy()
    ref = oracle.sgemm_rows(np.ascontiguousarray(Ast[:, :K]), np.ascontiguousarray(Bst[:, :N]))
    assert np.array_equal(Cst[:, :N].astype(np.float64), ref)          # integer inputs: exact
    # (columns N..ldc-1 of a W buffer are undefined after execute: W args are
    # not uploaded, include/jacc.h)
    A0 = np.zeros((5, 0), np.float32); B0 = np.zeros((0, 7), np.float32); C0 = np.full((5, 7), 3.0, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_SGEMM_F32, [g.a(A0, R), g.a(B0, R), g.a(C0, W)],
               jacc.jacc_sgemm_params_t(5, 7, 0, 0, 7, 7, mode, 0))
    g.run(); g.destroy()
    assert np.all(C0 == 0.0)


@pytest.mark.parametrize("mode", [J.JACC_SGEMM_FFMA, J.JACC_SGEMM_3XTF32], ids=["ffma", "3xtf32"])
@pytest.mark.parametrize("shape", SG_SHAPES)
def test_sgemm_gates(mode, shape):
    M, N, K = shape
    A, B = synth.sgemm_inputs(M, N, K, "int", seed=M + N + K)
    C = _sgemm(A, B, mode)
    assert np.array_equal(C.astype(np.float64), oracle.sgemm_rows(A, B)), "integer inputs must be exact"
    A, B = synth.sgemm_inputs(M, N, K, "unit", seed=M * 3 + K)
    C = _sgemm(A, B, mode).astype(np.float64)
    Ro = oracle.sgemm_rows(A, B)
    assert np.max(np.abs(C - Ro) / np.maximum(np.abs(Ro), 1e-30)) <= 1e-4
    A, B = synth.sgemm_inputs(M, N, K, "signed", seed=M * 5 + N)
    C = _sgemm(A, B, mode).astype(np.float64)
    Ro = oracle.sgemm_rows(A, B)
    assert np.linalg.norm(C - Ro) <= 1e-4 * np.linalg.norm(Ro)
    AB = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    assert np.all(np.abs(C - Ro) <= 1e-4 * AB + 1e-30)


@pytest.mark.slow
@pytest.mark.parametrize("dist", ["unit", "signed"])
def test_sgemm_full_size_config4_elementwise(dist):
    """8192^3 (BASELINE config 4), EVERY element against the full fp64 oracle:
    U[0,1) gate M1 (elementwise relative 1e-4); U[-1,1) gate M2 (normwise
    1e-4 and componentwise 1e-4 (|A||B|)), plus Freivalds on the whole C."""
    n = synth.CFG4_MNK
    A, B = synth.sgemm_inputs(n, n, n, dist)
    C = _sgemm(A, B, J.JACC_SGEMM_3XTF32, device_args=True).astype(np.float64)
    Ro = oracle.sgemm_rows(A, B)
    if dist == "unit":
        assert np.max(np.abs(C - Ro) / np.abs(Ro)) <= 1e-4
    else:
        assert np.linalg.norm(C - Ro) <= 1e-4 * np.linalg.norm(Ro)
        # |A||B| is a GEMM of non-negative inputs: the oracle computes it too
        AB = oracle.sgemm_rows(np.abs(A), np.abs(B))
        assert np.all(np.abs(C - Ro) <= 1e-4 * AB)
    del Ro
    x = synth.rng(8).standard_normal(n)
    lhs = C @ x
    rhs = A.astype(np.float64) @ (B.astype(np.float64) @ x)
    bound = np.abs(A).astype(np.float64) @ (np.abs(B).astype(np.float64) @ np.abs(x))
    assert np.all(np.abs(lhs - rhs) <= 1e-4 * bound)


# ----------------------------------------------------------------- N-body
def _nbody_graph(pos, vel, steps, dt=synth.NBODY_DT, eps2=synth.NBODY_EPS2, G=synth.NBODY_G):
    n = pos.shape[0]
    P = [pos.copy(), np.zeros_like(pos)]
    V = vel.copy()
    g = _graph()
    for k in range(steps):
        g.add_task(J.JACC_OP_NBODY_STEP_F32,
                   [g.a(P[k % 2], R, True, f32x4=True), g.a(V, RW, True, f32x4=True),
                    g.a(P[(k + 1) % 2], W, True, f32x4=True)],
                   jacc.jacc_nbody_params_t(0, dt, eps2, G))
    g.run()
    st = g.stats()
    g.destroy()
    return P[steps % 2], V, st


@pytest.mark.parametrize("n,steps", [(1, 1), (7, 3), (1000, 1), (4096, 10)])
def test_nbody_steps(n, steps):
    pos, vel = synth.nbody_state(n, seed=100 + n)
    gp, gv, st = _nbody_graph(pos, vel, steps)
    op, ov = oracle.nbody_steps(pos, vel, steps)
    assert np.max(np.abs(gp[:, :3] - op[:, :3])) <= 1e-4 * 1.0
    vs = max(np.mean(np.linalg.norm(ov[:, :3], axis=1)), 1e-30)
    assert np.max(np.abs(gv[:, :3] - ov[:, :3])) <= 1e-4 * vs
    assert np.array_equal(gp[:, 3], pos[:, 3])
    if steps > 1:   # SURVEY count table: 10 chained steps -> 2 H2D + 3 D2H
        assert (st["h2d_count"], st["d2h_count"]) == (2, 3)


@pytest.mark.parametrize("case", ["mixed", "one_tile_mixed"])
def test_nbody_unequal_masses(case):
    """The kernel's general (per-source mass) tile path: masses that differ
    across the whole set, or in one 256-source tile only (that tile takes
    the general path, the others the equal-mass path)."""
    n, steps = 5000, 3
    pos, vel = synth.nbody_state(n, seed=77)
    if case == "mixed":
        pos[:, 3] = (synth.uniform_f32(n, 78, 0.5, 1.5) / n).astype(np.float32)
    else:
        pos[300, 3] = np.float32(3.0 / n)
    gp, gv, _ = _nbody_graph(pos, vel, steps)
    op, ov = oracle.nbody_steps(pos, vel, steps)
    assert np.max(np.abs(gp[:, :3] - op[:, :3])) <= 1e-4
    vs = np.mean(np.linalg.norm(ov[:, :3], axis=1))
    assert np.max(np.abs(gv[:, :3] - ov[:, :3])) <= 1e-4 * vs


def test_nbody_full_size_mixed_masses_and_kernel_variants():
    """2^17 bodies: the full grid takes the single-buffered kernel (many
    waves), a 1/2 target shard the double-buffered one, 1/4 and 1/8 shards the
    mixed grid (3-pair units, then 1-pair units for the last wave) -- with
    unequal masses (general tile path) the sampled accelerations match the
    oracle, and every shard is bitwise equal to the full run's slice (the
    same chunk and tile grouping in every variant)."""
    n = synth.CFG5_N
    pos, vel = synth.nbody_state(n, seed=81)
    pos[:, 3] = (synth.uniform_f32(n, 82, 0.5, 1.5) / n).astype(np.float32)
    prm = lambda lo: jacc.jacc_nbody_params_t(lo, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G)
    dpos = _dev(pos)

    def step(lo, hi):
        dv = _dev(vel[lo:hi]); out = torch.zeros_like(dv)
        g = _graph()
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(dpos, R, f32x4=True), g.a(dv, RW, f32x4=True),
                                               g.a(out, W, f32x4=True)], prm(lo))
        g.run(); g.destroy()
        return dv.cpu().numpy(), out.cpu().numpy()
    full_v, full_p = step(0, n)
    idx = np.concatenate([synth.rng(83).integers(0, n, 48), [0, n - 1]])
    a_ref = oracle.nbody_accel(pos.astype(np.float64), idx)
    a_gpu = full_v[idx, :3].astype(np.float64) / synth.NBODY_DT
    assert np.max(np.linalg.norm(a_gpu - a_ref, axis=1) / np.linalg.norm(a_ref, axis=1)) <= 1e-4
    for k, r in ((2, 1), (4, 2), (8, 5)):
        lo, hi = synth.shard_range(n, r, k)
        v, p = step(lo, hi)
        assert np.array_equal(v, full_v[lo:hi]) and np.array_equal(p, full_p[lo:hi]), (k, r)


def test_nbody_mass_scaling_exact():
    """a is linear in the masses; doubling every mass (a power of two) must
    double the step's velocity change bit for bit, on both tile paths."""
    n = 3000
    pos, vel = synth.nbody_state(n, seed=79)
    outs = []
    for scale in (1.0, 2.0):
        for mixed in (False, True):
            p = pos.copy()
            p[:, 3] = np.float32(2.0 ** -12) * np.float32(scale)
            if mixed:
                p[::7, 3] *= np.float32(0.5)
            _, gv, _ = _nbody_graph(p, vel, 1)
            outs.append(gv[:, :3].copy())
    assert np.array_equal(outs[2], 2 * outs[0])
    assert np.array_equal(outs[3], 2 * outs[1])


def test_nbody_full_size_one_step_sampled_and_momentum():
    n = synth.CFG5_N
    pos, vel = synth.nbody_state(n)
    dP = [_dev(pos), torch.zeros_like(_dev(pos))]
    dV = _dev(vel)
    g = _graph()
    for k in range(synth.CFG5_STEPS):
        g.add_task(J.JACC_OP_NBODY_STEP_F32,
                   [g.a(dP[k % 2], R, f32x4=True), g.a(dV, RW, f32x4=True), g.a(dP[(k + 1) % 2], W, f32x4=True)],
                   jacc.jacc_nbody_params_t(0, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G))
        if k == 0:
            pass
    g.run()
    v10 = dV.cpu().numpy().astype(np.float64)
    m = pos[:, 3:4].astype(np.float64)
    P10 = np.sum(m * v10[:, :3], axis=0)
    assert np.max(np.abs(P10)) <= 1e-5 * np.sum(m * np.abs(v10[:, :3]))   # momentum conserved
    g.destroy()
    # one step, sampled bodies: recover a_i from v_1 = a_i dt (v_0 = 0)
    dV = _dev(vel); out = torch.zeros_like(dV)
    g = _graph()
    g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(_dev(pos), R, f32x4=True), g.a(dV, RW, f32x4=True),
                                           g.a(out, W, f32x4=True)],
               jacc.jacc_nbody_params_t(0, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G))
    g.run()
    idx = np.concatenate([synth.rng(3).integers(0, n, 64), [0, n - 1]])
    a_ref = oracle.nbody_accel(pos.astype(np.float64), idx)
    a_gpu = dV.cpu().numpy()[idx, :3].astype(np.float64) / synth.NBODY_DT
    rel = np.linalg.norm(a_gpu - a_ref, axis=1) / np.linalg.norm(a_ref, axis=1)
    assert np.max(rel) <= 1e-4
    g.destroy()


def test_nbody_shard_invariance_bitwise():
    n, P = 3000, 4
    pos, vel = synth.nbody_state(n, seed=5)
    vel[:, :3] = synth.rng(6).standard_normal((n, 3)).astype(np.float32) * 0.1
    full_v = vel.copy(); full_p = np.zeros_like(pos)
    g = _graph()
    g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(pos, R, f32x4=True), g.a(full_v, RW, f32x4=True),
                                           g.a(full_p, W, f32x4=True)], jacc.jacc_nbody_params_t(0, 0.016, 0.01, 1.0))
    g.run(); g.destroy()
    for r in range(P):
        lo, hi = synth.shard_range(n, r, P)
        v = vel[lo:hi].copy(); p = np.zeros_like(v)
        g = _graph()
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(pos, R, f32x4=True), g.a(v, RW, f32x4=True),
                                               g.a(p, W, f32x4=True)], jacc.jacc_nbody_params_t(lo, 0.016, 0.01, 1.0))
        g.run(); g.destroy()
        assert np.array_equal(v, full_v[lo:hi]) and np.array_equal(p, full_p[lo:hi])


_V1_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import synth, torch
import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
from paper_1508_06791_b200.torch_glue import make_graph
M, N, K, seed = map(int, sys.argv[2:6])
A, B = synth.sgemm_inputs(M, N, K, "signed", seed=seed)
C = np.zeros((M, N), np.float32)
g, _ = make_graph(0)
g.add_task(J.JACC_OP_SGEMM_F32, [g.a(A, 1), g.a(B, 1), g.a(C, 2)],
           jacc.jacc_sgemm_params_t(M, N, K, K, N, N, J.JACC_SGEMM_3XTF32, 0))
g.run(); g.destroy()
np.save(sys.argv[6], C)
"""


@pytest.mark.parametrize("shape", [(256, 256, 256), (300, 520, 1000), (1000, 1000, 4096), (2048, 2048, 1024)])
def test_sgemm_inkernel_split_bitwise_equals_presplit(shape, tmp_path):
    """The default path feeds the RAW fp32 tiles to kind::tf32 as the hi
    operand (the tensor core reads only the TF32 bits) and splits lo inside
    the kernel; the pre-split path (JACC_SGEMM_V1=1) writes x_hi = x &
    0xFFFFE000 and x_lo = x - x_hi to memory first.  Both issue the same
    three MMAs in the same order, so they agree BIT FOR BIT exactly when the
    hardware's operand read is that truncation -- which this pins."""
    import os
    import subprocess
    import sys
    M, N, K = shape
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for v1 in ("0", "1"):
        f = str(tmp_path / f"c{v1}.npy")
        env = dict(os.environ, JACC_SGEMM_V1=v1)
        r = subprocess.run([sys.executable, "-c", _V1_SCRIPT, root, str(M), str(N), str(K), "77", f],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs[v1] = np.load(f)
    assert np.array_equal(outs["0"].view(np.uint32), outs["1"].view(np.uint32))
    A, B = synth.sgemm_inputs(M, N, K, "signed", seed=77)
    Ro = oracle.sgemm_rows(A, B)
    assert np.linalg.norm(outs["0"] - Ro) <= 1e-4 * np.linalg.norm(Ro)
