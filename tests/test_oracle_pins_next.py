"""Pins for the oracle functions of the SURVEY §8(f) NEXT rows (CPU only)."""
import numpy as np
import pytest
from scipy.signal import convolve2d

import oracle
import synth


# ------------------------------------------------------------- f1: conv2d
def test_conv2d_delta_gives_flipped_placement(orc):
    # a unit impulse at (y0, x0) reproduces the filter: out[y0 + i - r][x0 + j - r] = f[i][j]
    f = synth.rng(1).random((5, 5), dtype=np.float32)
    img = np.zeros((16, 20), np.float32)
    img[7, 9] = 1.0
    out, _ = orc.conv2d(img, f)
    for i in range(5):
        for j in range(5):
            assert out[7 + i - 2, 9 + j - 2] == f[i, j]
    assert np.count_nonzero(out) == 25


def test_conv2d_box_filter_closed_form(orc):
    img = np.full((9, 11), 3.0, np.float32)
    out, _ = orc.conv2d(img, np.ones((5, 5), np.float32))
    assert out[4, 5] == 75.0          # interior: 25 taps
    assert out[0, 0] == 27.0          # corner: 3 x 3 taps inside
    assert out[0, 5] == 45.0          # edge: 3 x 5 taps
    assert out[1, 1] == 48.0          # 4 x 4 taps


def test_conv2d_vs_scipy_and_separable(orc):
    img = synth.uniform_f32(37 * 53, 4, -1, 1).reshape(37, 53)
    f = synth.uniform_f32(25, 5, -1, 1).reshape(5, 5)
    out, ab = orc.conv2d(img, f)
    ref = convolve2d(img.astype(np.float64), f.astype(np.float64), mode="same", boundary="fill")
    assert np.max(np.abs(out - ref)) <= 1e-12 * np.max(ab)
    u = np.array([1, 2, 3, 2, 1], np.float32); v = np.array([-1, 0, 2, 0, 1], np.float32)
    out, _ = orc.conv2d(img, np.outer(u, v))
    rows = np.array([np.convolve(r.astype(np.float64), v, mode="same") for r in img])
    sep = np.array([np.convolve(c, u, mode="same") for c in rows.T]).T
    assert np.max(np.abs(out - sep)) <= 1e-12 * np.max(np.abs(sep))


def test_conv2d_linearity_and_scale(orc):
    a = synth.uniform_f32(24 * 24, 6).reshape(24, 24)
    b = synth.uniform_f32(24 * 24, 7).reshape(24, 24)
    f = synth.uniform_f32(9, 8).reshape(3, 3)
    oa, _ = orc.conv2d(a, f); ob, _ = orc.conv2d(b, f)
    oab, ab = orc.conv2d((a + b).astype(np.float32), f)
    assert np.max(np.abs(oab - (oa + ob))) <= 1e-6 * np.max(ab)
    _, absum = orc.conv2d(np.abs(a), np.abs(f))
    assert np.all(ab >= 0)


# ------------------------------------------------- f3: correlation matrix
def test_corr_spec_example_and_brute_force(orc):
    # bitsets 0b1011 and 0b1110 -> intersection count popc(0b1010) = 2
    A = np.array([[0b1011], [0b1110]], np.uint32)
    C = orc.corr_popc(A)
    assert C[0, 1] == 2 and C[1, 0] == 2 and C[0, 0] == 3 and C[1, 1] == 3
    A = synth.corr_bitsets(7, 96, 0.3, seed=4)
    B = synth.corr_bitsets(5, 96, 0.6, seed=5)
    C = orc.corr_popc(A, B)
    for i in range(7):
        for j in range(5):   # python big-int bit counting
            assert C[i, j] == sum(bin(int(a) & int(b)).count("1") for a, b in zip(A[i], B[j]))


def test_corr_invariants(orc):
    A = synth.corr_bitsets(64, 1024, 0.5, seed=6)
    C = orc.corr_popc(A)
    assert np.array_equal(C, C.T)
    assert np.array_equal(np.diag(C), np.unpackbits(A.view(np.uint8), axis=1).sum(axis=1))
    ones = np.full((3, 4), 0xFFFFFFFF, np.uint32)
    assert np.all(orc.corr_popc(ones) == 128)
    assert np.all(orc.corr_popc(ones, np.zeros((2, 4), np.uint32)) == 0)
    # counts against documents unpacked by numpy: C = X X^T for the 0/1 matrix X
    X = np.unpackbits(A.view(np.uint8), axis=1, bitorder="little").astype(np.int64)
    assert np.array_equal(C, X @ X.T)


# ------------------------------------------------------------- f4: SpMV
def test_spmv_vs_scipy_and_closed_forms(orc):
    from scipy.sparse import csr_matrix
    rp, col, val = synth.banded_csr(500, 11000, bandwidth=40, seed=3)
    x = synth.uniform_f32(500, 9, -1, 1)
    y, ab = orc.spmv_csr(rp, col, val, x)
    A = csr_matrix((val.astype(np.float64), col, rp), shape=(500, 500))
    assert np.max(np.abs(y - A @ x.astype(np.float64))) <= 1e-12 * np.max(ab)
    # x = ones: row sums; identity matrix: y = x
    y1, _ = orc.spmv_csr(rp, col, val, np.ones(500, np.float32))
    assert np.allclose(y1, np.add.reduceat(val.astype(np.float64), rp[:-1]) * (np.diff(rp) > 0), rtol=0, atol=1e-12)
    I_rp = np.arange(501, dtype=np.int32); I_col = np.arange(500, dtype=np.int32)
    yi, _ = orc.spmv_csr(I_rp, I_col, np.ones(500, np.float32), x)
    assert np.array_equal(yi, x.astype(np.float64))
    # empty rows give 0
    rp0 = np.zeros(4, np.int32)
    y0, _ = orc.spmv_csr(rp0, np.zeros(0, np.int32), np.zeros(0, np.float32), np.ones(3, np.float32))
    assert np.array_equal(y0, np.zeros(3))


def test_banded_csr_is_symmetric_pattern_with_diagonal():
    rp, col, val = synth.banded_csr(300, 4000, bandwidth=20, seed=2)
    rows = np.repeat(np.arange(300), np.diff(rp))
    pattern = set(zip(rows.tolist(), col.tolist()))
    assert all((j, i) in pattern for i, j in pattern)
    assert all((i, i) in pattern for i in range(300))


# --------------------------------------------- halo bands (f1 row sharding)
@pytest.mark.parametrize("H,P,r", [(37, 2, 2), (40, 4, 2), (9, 3, 1), (50, 8, 4)])
def test_halo_band_pins(H, P, r):
    """oracle.halo_band: the bands' middle rows tile the image; a band's top
    halo is the previous band's last r rows (zeros above row 0), its bottom
    halo the next band's first r rows (zeros below the last row); and the
    convolution of every extended band, middle rows, reassembles the
    whole-image convolution exactly (each output row reads only rows within
    r of it)."""
    import synth
    img = synth.uniform_f32(H * 13, 90 + H, -1, 1).reshape(H, 13)
    f = synth.uniform_f32((2 * r + 1) ** 2, 91, -1, 1).reshape(2 * r + 1, 2 * r + 1)
    full, _ = oracle.conv2d(img, f)
    mids, outs = [], []
    for q in range(P):
        lo, hi = synth.shard_range(H, q, P)
        ext = oracle.halo_band(img, lo, hi, r)
        assert ext.shape == (hi - lo + 2 * r, 13)
        mids.append(ext[r:r + hi - lo])
        top, bot = ext[:r], ext[r + hi - lo:]
        if q == 0:
            assert not top.any()
        else:
            plo, phi = synth.shard_range(H, q - 1, P)
            assert np.array_equal(top, img[phi - r:phi])
        if q == P - 1:
            assert not bot.any()
        else:
            assert np.array_equal(bot, img[hi:hi + r])
        o, _ = oracle.conv2d(ext, f)
        outs.append(o[r:r + hi - lo])
    assert np.array_equal(np.concatenate(mids), img)
    assert np.array_equal(np.concatenate(outs), full)
