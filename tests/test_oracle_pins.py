"""Pins for the CPU oracle (oracle/jacc_oracle.c) -- CPU only.

Each test ties an oracle function to something OTHER than itself: a closed
form, a brute-force count, a conservation law or symmetry of the mathematics,
a worked example from tests/golden/ (cited), or an independent library
routine (numpy / scipy / math).  A plausible mistake in the oracle (a dropped
term, a wrong sign or index, a transposed operand) fails at least one.
"""
import json
import math
import os

import numpy as np
import pytest
from scipy.special import ndtr

import synth

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ vector add
def test_vadd_closed_form(orc):
    n = 1 << 20
    a = np.arange(n, dtype=np.float32)
    b = (n - np.arange(n)).astype(np.float32)
    c = orc.vadd(a, b)
    assert np.all(c == np.float32(n))


def test_vadd_matches_ieee_fp32_add(orc):
    a, b = synth.vadd_inputs(1 << 16)
    a[:4] = [np.inf, -np.inf, 1e38, np.float32(0.1)]
    b[:4] = [-np.inf, 1.0, 1e38, np.float32(0.2)]
    c = orc.vadd(a, b)
    ref = a + b   # numpy float32 add: one RN binary32 add
    assert np.array_equal(c.view(np.uint32)[1:], ref.view(np.uint32)[1:])
    assert np.isnan(c[0])


# ------------------------------------------------------------------- reduction
def test_reduce_gauss(orc):
    n = 1 << 20
    x = np.arange(1, n + 1, dtype=np.float32)   # exact in fp32 (n <= 2^24)
    s, a = orc.reduce_sum(x)
    assert s == n * (n + 1) // 2
    assert a == s


def test_reduce_golden(orc):
    g = GOLDEN["reduce_1_to_1024"]
    s, _ = orc.reduce_sum(np.arange(1, g["n"] + 1, dtype=np.float32))
    assert s == g["expected"]
    g = GOLDEN["reduce_all_ones_65536"]
    s, _ = orc.reduce_sum(np.ones(g["n"], np.float32))
    assert s == g["expected"]


def test_reduce_empty_and_init(orc):
    assert orc.reduce_sum(np.zeros(0, np.float32)) == (0.0, 0.0)
    s, _ = orc.reduce_sum(np.ones(10, np.float32), init=2.5)
    assert s == 12.5


def test_reduce_vs_fsum_signed(orc):
    x = synth.uniform_f32(1 << 18, 7, -1.0, 1.0)
    s, a = orc.reduce_sum(x)
    ref = math.fsum(float(v) for v in x)
    assert abs(s - ref) <= 1e-12 * a
    assert abs(a - math.fsum(abs(float(v)) for v in x)) <= 1e-12 * a


# ------------------------------------------------------------------- histogram
def test_hist_brute_force(orc):
    keys = synth.hist_keys(3000, 256, seed=3, dist="with_out_of_range")
    bins = orc.histogram(keys, 256)
    kl = keys.tolist()
    for k in range(256):
        assert bins[k] == sum(1 for v in kl if v == k)


def test_hist_closed_forms(orc):
    n = 1 << 16
    bins = orc.histogram(np.arange(n, dtype=np.int32) % 256, 256)
    assert np.all(bins == n // 256)
    bins = orc.histogram(np.full(n, 17, np.int32), 256)
    assert bins[17] == n and bins.sum() == n
    g = GOLDEN["histogram_0_to_255_once"]
    bins = orc.histogram(np.arange(256, dtype=np.int32), g["nbins"])
    assert np.all(bins == g["expected_each"])


def test_hist_sum_and_bincount(orc):
    keys = synth.hist_keys(1 << 20, 256, seed=5, dist="with_out_of_range")
    bins = orc.histogram(keys, 256)
    inr = keys[(keys >= 0) & (keys < 256)]
    assert bins.sum() == inr.size
    assert np.array_equal(bins, np.bincount(inr, minlength=256))


def test_hist_accumulate(orc):
    keys = synth.hist_keys(1000, 64, seed=9)
    init = np.arange(64, dtype=np.int32)
    bins = orc.histogram(keys, 64, init=init)
    assert np.array_equal(bins - init, np.bincount(keys, minlength=64))
    g = GOLDEN["atomic_1024_adds"]
    assert orc.histogram(np.zeros(g["n"], np.int32), 1)[0] == g["expected"]


# ---------------------------------------------------------------- Black-Scholes
def _bs_exact(S, K, T, R, sig):
    d1 = (math.log(S / K) + (R + sig * sig / 2) * T) / (sig * math.sqrt(T))
    d2 = d1 - sig * math.sqrt(T)
    call = S * ndtr(d1) - K * math.exp(-R * T) * ndtr(d2)
    put = K * math.exp(-R * T) * ndtr(-d2) - S * ndtr(-d1)
    return call, put


def test_phi_vs_ndtr_within_AS_bound(orc):
    # Abramowitz & Stegun 26.2.17: |error| < 7.5e-8
    for x in np.linspace(-8, 8, 4001):
        assert abs(orc.bs_phi(x) - ndtr(x)) < 7.6e-8
    assert orc.bs_phi(0.0) == pytest.approx(0.5, abs=7.5e-8)
    assert orc.bs_phi(-1.0) + orc.bs_phi(1.0) == pytest.approx(1.0, abs=1e-15)


def test_bs_textbook_golden(orc):
    g = GOLDEN["blackscholes_textbook"]
    c, p = orc.bs_price(g["S"], g["K"], g["T"], g["R"], g["sigma"])
    scale = g["S"] + g["K"] * math.exp(-g["R"] * g["T"])
    assert abs(c - g["call_exact"]) <= scale * 7.5e-8
    assert abs(p - g["put_exact"]) <= scale * 7.5e-8
    assert abs(c - g["call_approx"]) <= g["abs_tol_call_approx"]
    ce, pe = _bs_exact(g["S"], g["K"], g["T"], g["R"], g["sigma"])
    assert ce == pytest.approx(g["call_exact"], abs=1e-9)


def test_bs_put_call_parity_and_exact(orc):
    rng = np.random.default_rng(11)
    n = 2000
    S = rng.uniform(5, 150, n).astype(np.float32)
    K = rng.uniform(5, 150, n).astype(np.float32)
    T = rng.uniform(0.1, 10, n).astype(np.float32)
    R = rng.uniform(0.0, 0.1, n).astype(np.float32)
    V = rng.uniform(0.01, 0.8, n).astype(np.float32)
    call, put = orc.blackscholes_soa(S, K, T, R, V)
    for i in range(0, n, 7):
        s, k, t, r, v = (float(z[i]) for z in (S, K, T, R, V))
        scale = s + k * math.exp(-r * t)
        # parity holds exactly in real arithmetic since phi(-x) = 1 - phi(x)
        assert abs((call[i] - put[i]) - (s - k * math.exp(-r * t))) <= 1e-12 * scale
        ce, pe = _bs_exact(s, k, t, r, v)
        assert abs(call[i] - ce) <= 1.6e-7 * scale
        assert abs(put[i] - pe) <= 1.6e-7 * scale


def test_bs_monotone_and_limits(orc):
    S = np.linspace(20, 200, 50).astype(np.float32)
    one = np.ones_like(S)
    call, put = orc.blackscholes_soa(S, 100 * one, one, 0.05 * one, 0.2 * one)
    assert np.all(np.diff(call) > 0) and np.all(np.diff(put) < 0)
    c, p = orc.bs_price(1000.0, 10.0, 1.0, 0.05, 0.2)   # deep in the money
    assert c == pytest.approx(1000.0 - 10.0 * math.exp(-0.05), rel=1e-9)
    assert abs(p) < 1e-9


def test_bs_aparapi_mapping(orc):
    # X = X_lo u + X_hi (1-u): u=0 -> upper limits, u=1 -> lower limits
    assert orc.bs_params(0.0) == pytest.approx((100.0, 100.0, 10.0, 0.05, 0.10))
    assert orc.bs_params(1.0) == pytest.approx((10.0, 10.0, 1.0, 0.01, 0.01))
    u = synth.bs_rand(4096)
    call, put = orc.blackscholes(u)
    for i in range(0, 4096, 97):
        S, K, T, R, V = orc.bs_params(float(u[i]))
        c, p = orc.bs_price(S, K, T, R, V)
        assert (call[i], put[i]) == (c, p)
        ce, pe = _bs_exact(S, K, T, R, V)
        assert abs(call[i] - ce) <= 1.6e-7 * (S + K * math.exp(-R * T))


# ------------------------------------------------------------------------ SGEMM
def test_sgemm_integer_exact(orc):
    A, B = synth.sgemm_inputs(67, 45, 129, dist="int")
    C = orc.sgemm_rows(A, B)
    exact = A.astype(np.int64) @ B.astype(np.int64)   # exact integer arithmetic
    assert np.array_equal(C, exact.astype(np.float64))


def test_sgemm_identity_golden(orc):
    n = GOLDEN["sgemm_identity_8x8"]["n"]
    A, _ = synth.sgemm_inputs(n, n, n)
    C = orc.sgemm_rows(A, np.eye(n, dtype=np.float32))
    assert np.array_equal(C, A.astype(np.float64))
    C = orc.sgemm_rows(np.eye(n, dtype=np.float32), A)
    assert np.array_equal(C, A.astype(np.float64))


def test_sgemm_vs_numpy_and_transpose(orc):
    A, B = synth.sgemm_inputs(96, 80, 112, dist="signed")
    C = orc.sgemm_rows(A, B)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert np.max(np.abs(C - ref)) <= 1e-12 * np.max(np.abs(A).astype(np.float64) @ np.abs(B))
    Ct = orc.sgemm_rows(np.ascontiguousarray(B.T), np.ascontiguousarray(A.T))
    assert np.max(np.abs(Ct.T - C)) <= 1e-12 * np.max(np.abs(C))
    rows = np.array([0, 5, 95, 40], np.int64)
    assert np.array_equal(orc.sgemm_rows(A, B, rows), C[rows])


def test_sgemm_freivalds(orc):
    A, B = synth.sgemm_inputs(256, 192, 320, dist="signed")
    C = orc.sgemm_rows(A, B)
    x = np.random.default_rng(2).standard_normal(192)
    lhs = C @ x
    rhs = A.astype(np.float64) @ (B.astype(np.float64) @ x)
    bound = np.abs(A).astype(np.float64) @ (np.abs(B).astype(np.float64) @ np.abs(x))
    assert np.all(np.abs(lhs - rhs) <= 1e-12 * bound)


# ----------------------------------------------------------------------- N-body
def test_nbody_two_body_closed_form(orc):
    r, m1, m2, eps2, G = 0.7, 0.3, 0.5, 0.01, 1.7
    pos = np.array([[0, 0, 0, m1], [r, 0, 0, m2]], np.float64)
    a = orc.nbody_accel(pos, eps2=eps2, G=G)
    f = r / (r * r + eps2) ** 1.5
    assert a[0] == pytest.approx([G * m2 * f, 0, 0], rel=1e-14)
    assert a[1] == pytest.approx([-G * m1 * f, 0, 0], rel=1e-14)


def test_nbody_cube_symmetry(orc):
    verts = np.array([[x, y, z, 1.0] for x in (-1, 1) for y in (-1, 1) for z in (-1, 1)], float)
    pos = np.vstack([verts, [[0, 0, 0, 2.0]]])
    a = orc.nbody_accel(pos, eps2=0.01, G=1.0)
    assert np.max(np.abs(a[8])) < 1e-15
    mags = np.linalg.norm(a[:8], axis=1)
    assert np.allclose(mags, mags[0], rtol=1e-14)
    for i in range(8):   # pulled toward the centre, along -x_i
        unit = pos[i, :3] / np.linalg.norm(pos[i, :3])
        assert np.allclose(a[i] / mags[i], -unit, atol=1e-14)


def test_nbody_third_law_linearity_translation(orc):
    pos, _ = synth.nbody_state(300, seed=8)
    pos = pos.astype(np.float64)
    pos[:, 3] = np.random.default_rng(3).uniform(0.5, 2.0, 300) / 300
    a = orc.nbody_accel(pos)
    m = pos[:, 3:4]
    scale = np.sum(m * np.abs(a))
    assert np.max(np.abs(np.sum(m * a, axis=0))) <= 1e-14 * scale
    a2 = orc.nbody_accel(pos, G=2.0)
    assert np.allclose(a2, 2 * a, rtol=1e-15, atol=0)
    sh = pos.copy(); sh[:, :3] += [0.25, -0.5, 0.125]
    assert np.allclose(orc.nbody_accel(sh), a, rtol=0, atol=1e-12 * np.max(np.abs(a)))
    tg = np.array([3, 299, 0, 150])
    assert np.array_equal(orc.nbody_accel(pos, tg), a[tg])


def test_nbody_steps_from_rest_and_momentum(orc):
    pos, vel = synth.nbody_state(256, seed=4)
    dt = 0.016
    a0 = orc.nbody_accel(pos.astype(np.float64))
    p1, v1 = orc.nbody_steps(pos, vel, 1, dt=dt)
    # symplectic Euler from rest: v1 = a0 dt, x1 = x0 + a0 dt^2
    assert np.allclose(v1[:, :3], a0 * dt, rtol=1e-15, atol=0)
    assert np.allclose(p1[:, :3], pos[:, :3].astype(np.float64) + a0 * dt * dt, rtol=0, atol=1e-15)
    assert np.array_equal(p1[:, 3], pos[:, 3].astype(np.float64))
    vel = vel.copy(); vel[:, :3] = np.random.default_rng(5).standard_normal((256, 3)) * 0.1
    p10, v10 = orc.nbody_steps(pos, vel, 10, dt=dt)
    m = pos[:, 3:4].astype(np.float64)
    P0 = np.sum(m * vel[:, :3], axis=0)
    P10 = np.sum(m * v10[:, :3], axis=0)
    assert np.max(np.abs(P10 - P0)) <= 1e-12 * np.sum(m * np.abs(v10[:, :3]))
