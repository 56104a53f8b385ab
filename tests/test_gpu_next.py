"""GPU parity for the SURVEY §8(f) NEXT rows, through the C-ABI."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
J = pytest.importorskip("paper_1508_06791_b200")
from paper_1508_06791_b200 import jacc  # noqa: E402
from paper_1508_06791_b200.torch_glue import make_graph  # noqa: E402

R, W = J.JACC_READ, J.JACC_WRITE


def _conv(img, f):
    H, Wd = img.shape
    k = f.shape[0]
    out = np.zeros_like(img)
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img, R), g.a(f, R), g.a(out, W)],
               jacc.jacc_conv2d_params_t(H, Wd, k // 2, 0))
    g.run()
    g.destroy()
    return out


def test_conv2d_misaligned_device_output():
    """A caller-owned DEVICE output that is only 4-byte aligned (a view at an
    odd element offset) must not reach the TMA kernel's 8-byte stores: it
    takes the simple kernel, same results."""
    import torch
    h, w = 64, 256
    img = synth.uniform_f32(h * w, 601, -1, 1).reshape(h, w)
    f = synth.uniform_f32(25, 602, -1, 1).reshape(5, 5)
    buf = torch.zeros(h * w + 1, device="cuda")
    out = buf[1:].view(h, w)
    assert out.data_ptr() % 8 == 4
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_CONV2D_F32, [g.a(torch.from_numpy(img).cuda(), R), g.a(torch.from_numpy(f).cuda(), R),
                                      g.a(out, W)], jacc.jacc_conv2d_params_t(h, w, 2, 0))
    g.run()
    g.destroy()
    ref, ab = oracle.conv2d(img, f)
    assert np.all(np.abs(out.cpu().numpy().astype(np.float64) - ref) <= 1e-5 * ab + 1e-30)


# TMA path: W % 4 == 0 and r == 2 (ragged 64 x 64 tiles, tiny images, many
# tiles per persistent block; 4739 x 4100 takes the 128 x 64 tile config,
# >= 16 tiles per SM, with ragged tiles on both edges); the others take the
# simple kernel
@pytest.mark.parametrize("H,Wd,r", [(1, 1, 2), (7, 9, 2), (33, 65, 1), (256, 256, 2), (100, 37, 3),
                                    (64, 64, 4), (2048, 2048, 2), (1, 4, 2), (3, 8, 1), (97, 132, 2),
                                    (33, 68, 1), (31, 260, 2), (1000, 1028, 2), (4739, 4100, 2)])
def test_conv2d_tolerance(H, Wd, r):
    img = synth.uniform_f32(H * Wd, 100 + H, -1, 1).reshape(H, Wd)
    f = synth.uniform_f32((2 * r + 1) ** 2, 200 + r, -1, 1).reshape(2 * r + 1, 2 * r + 1)
    out = _conv(img, f)
    ref, ab = oracle.conv2d(img, f)
    # map: 1e-5 of the output's natural scale sum |f| |img|
    assert np.all(np.abs(out - ref) <= 1e-5 * ab + 1e-30)


# split-K counts of the 1-SM kernel (split-K summed over DSMEM, corr.cu): 1024^2 x 16384
# -> 4; (100, 70, 131072) -> 8 on one ragged tile; (1152, 768) -> 5; (1408,
# 512) -> 6; (1280, 512) -> 7; (2000, 260) -> 4 with ragged rows and columns;
# 16-bit split partials up to 511 K blocks per split, 32-bit beyond ((100, 70, 2^20): 1024)
@pytest.mark.parametrize("ta,tb,docs", [(1, 1, 32), (5, 7, 96), (100, 70, 1000 * 32 // 32 * 32),
                                        (1024, 1024, 16384), (100, 70, 131072), (1152, 768, 8192),
                                        (1408, 512, 8192), (1280, 512, 8192), (2000, 260, 8192),
                                        (700, 500, 4096), (100, 70, 1 << 20)])
def test_corr_bit_exact(ta, tb, docs):
    A = synth.corr_bitsets(ta, docs, 0.5, seed=ta)
    B = synth.corr_bitsets(tb, docs, 0.3, seed=tb + 1)
    C = np.zeros((ta, tb), np.int32)
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(A.view(np.int32), R), g.a(B.view(np.int32), R), g.a(C, W)],
               jacc.jacc_corr_params_t(ta, tb, docs // 32))
    g.run()
    g.destroy()
    assert np.array_equal(C, oracle.corr_popc(A, B))


# >= 2^18 rows take the row-block streaming kernel (incl. a ragged last block)
@pytest.mark.parametrize("n,nnz,bw", [(1, 1, 1), (100, 900, 10), (5000, 100000, 300),
                                      (synth.SPMV_N, synth.SPMV_NNZ, 1600), ((1 << 18) + 77, 23 * (1 << 18), 1600)])
def test_spmv_tolerance(n, nnz, bw):
    rp, col, val = synth.banded_csr(n, nnz, bandwidth=bw, seed=n)
    x = synth.uniform_f32(n, 5, -1, 1)
    y = np.zeros(n, np.float32)
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_SPMV_CSR_F32, [g.a(rp, R), g.a(col, R), g.a(val, R), g.a(x, R), g.a(y, W)],
               jacc.jacc_spmv_params_t(n, n))
    g.run()
    g.destroy()
    ref, ab = oracle.spmv_csr(rp, col, val, x)
    assert np.all(np.abs(y - ref) <= 1e-5 * ab + 1e-30)


def _spmv(rp, col, val, x, n):
    y = np.full(n, np.nan, np.float32)     # W output: every row must be written
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_SPMV_CSR_F32, [g.a(rp, R), g.a(col, R), g.a(val, R), g.a(x, R), g.a(y, W)],
               jacc.jacc_spmv_params_t(n, x.size))
    g.run()
    g.destroy()
    return y


# irregular rows (power-law lengths, ~1/3 empty, explicit long rows): the
# lane kernel (30000 rows, one row of 12000) and the row-block stream kernel
# (2^18 + 77 rows; the block holding a 6000-non-zero row exceeds the
# 4096-product shared buffer and takes the per-row global path; a 30000 row)
@pytest.mark.parametrize("n,mean,long_rows", [(30000, 12.0, ((17, 12000),)),
                                              ((1 << 18) + 77, 8.0, ((1000, 6000), (200000, 30000),
                                                                    ((1 << 18) + 76, 5000)))])
def test_spmv_irregular_rows(n, mean, long_rows):
    rp, col, val = synth.powerlaw_csr(n, mean, seed=n, long_rows=long_rows)
    assert np.sum(np.diff(rp) == 0) > n // 10
    x = synth.uniform_f32(n, 9, -1, 1)
    y = _spmv(rp, col, val, x, n)
    ref, ab = oracle.spmv_csr(rp, col, val, x)
    assert np.all(np.abs(y.astype(np.float64) - ref) <= 1e-5 * ab + 1e-30)
    assert np.all(y[np.diff(rp) == 0] == 0.0)       # empty rows: exactly 0


@pytest.mark.parametrize("n", [1, 1000, 1 << 18])
def test_spmv_all_rows_empty(n):
    rp = np.zeros(n + 1, np.int32)
    col = np.zeros(0, np.int32); val = np.zeros(0, np.float32)
    x = synth.uniform_f32(n, 10, -1, 1)
    y = _spmv(rp, col, val, x, n)
    assert np.all(y == 0.0)


@pytest.mark.parametrize("shape", [(40, 50), (40, 132), (4739, 4100)])   # simple kernel / TMA path (zero-filled halo)
def test_conv2d_delta_exact(shape):
    f = synth.uniform_f32(25, 3).reshape(5, 5)
    img = np.zeros(shape, np.float32)
    h, w = shape
    img[0, 0] = 1.0; img[20, 30] = 1.0; img[h - 1, w - 1] = 1.0; img[0, w - 1] = 1.0; img[h - 1, w // 2 - 5] = 1.0   # impulses >= 5 apart: responses never overlap
    out = _conv(img, f)
    ref, _ = oracle.conv2d(img, f)
    assert np.array_equal(out.astype(np.float64), ref)


@pytest.mark.slow
def test_conv2d_roofline_size_sampled_strips():
    """16384^2 (bench next_rows' roofline point, the TMA kernel): sampled
    32-row strips -- top edge, bottom edge, interior, ragged tile rows --
    against the fp64 oracle run on the strip plus its 2-row halos (rows whose
    5x5 window stays inside the strip equal the full-image result)."""
    import torch
    n, r = 16384, 2
    img = synth.uniform_f32(n * n, 501, -1, 1).reshape(n, n)
    f = synth.uniform_f32(25, 502, -1, 1).reshape(5, 5)
    dimg = torch.from_numpy(img).cuda()
    out = torch.empty_like(dimg)
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_CONV2D_F32, [g.a(dimg, R), g.a(torch.from_numpy(f).cuda(), R), g.a(out, W)],
               jacc.jacc_conv2d_params_t(n, n, r, 0))
    g.run()
    g.destroy()
    for y0 in (0, 64 * 37 + 5, 8191, n - 32):
        lo, hi = max(0, y0 - r), min(n, y0 + 32 + r)
        ref, ab = oracle.conv2d(img[lo:hi], f)
        got = out[y0:y0 + 32].cpu().numpy().astype(np.float64)
        ref, ab = ref[y0 - lo:y0 - lo + 32], ab[y0 - lo:y0 - lo + 32]
        assert np.all(np.abs(got - ref) <= 1e-5 * ab + 1e-30), y0


@pytest.mark.slow
def test_spmv_roofline_size_stream_kernel():
    """2M rows x 23 non-zeros (bench next_rows' roofline point, the row-block
    streaming kernel) against the fp64 oracle, every row."""
    n = 1 << 21
    rp, col, val = synth.banded_csr(n, 23 * n)
    x = synth.uniform_f32(n, 503, -1, 1)
    y = np.zeros(n, np.float32)
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_SPMV_CSR_F32, [g.a(rp, R), g.a(col, R), g.a(val, R), g.a(x, R), g.a(y, W)],
               jacc.jacc_spmv_params_t(n, n))
    g.run()
    g.destroy()
    ref, ab = oracle.spmv_csr(rp, col, val, x)
    assert np.all(np.abs(y.astype(np.float64) - ref) <= 1e-5 * ab + 1e-30)


@pytest.mark.parametrize("same", [True, False])
def test_corr_replayed_graph_bit_exact(same):
    """corr inside a captured plan (JACC_GRAPH_REPLAY): the GEMM is launched
    with programmatic stream serialization after the unpack kernel and a
    (1, 1, splits) cluster -- both must survive stream capture.  Replayed
    three times with new bitsets between runs (the host buffers are re-read
    every execute), each result bit-exact."""
    g, _ = make_graph(0, flags=J.JACC_GRAPH_REPLAY)
    A = synth.corr_bitsets(1024, 16384, 0.5, seed=11)
    B = A if same else synth.corr_bitsets(300, 16384, 0.3, seed=12)
    C = np.zeros((1024, B.shape[0]), np.int32)
    g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(A.view(np.int32), R), g.a(B.view(np.int32), R), g.a(C, W)],
               jacc.jacc_corr_params_t(1024, B.shape[0], 512))
    for it in range(3):
        if it:
            A[:] = synth.corr_bitsets(1024, 16384, 0.5, seed=11 + 7 * it)
            if not same:
                B[:] = synth.corr_bitsets(300, 16384, 0.3, seed=12 + 7 * it)
        g.run()
        assert np.array_equal(C, oracle.corr_popc(A, B)), it
    assert g.stats()["graph_replays"] >= 1
    g.destroy()


# ------------------------------------------- f1 row-band sharding (halo rows)
def _conv_band_graph(g, band, f, rows, Wd, r):
    """halo exchange of the band, then conv2d of the extended band."""
    ext = np.zeros((rows + 2 * r, Wd), np.float32)
    out = np.zeros((rows, Wd), np.float32)
    g.add_task(J.JACC_OP_HALO_EXCHANGE_F32, [g.a(band, R), g.a(ext, W)], jacc.jacc_halo_params_t(rows, Wd, r, 0))
    g.add_task(J.JACC_OP_CONV2D_F32, [g.a(ext, R), g.a(f, R), g.a(out, W)],
               jacc.jacc_conv2d_params_t(rows, Wd, r, J.JACC_CONV2D_HALO_ROWS))
    return ext, out


@pytest.mark.parametrize("shape,r", [((300, 256), 2), ((300, 250), 2), ((77, 64), 1), ((2048, 2048), 2), ((65, 40), 4)])
def test_conv2d_halo_rows_world1(shape, r):
    """World 1: the halo exchange gives [zeros][image][zeros] and the halo-row
    convolution equals the plain same-size convolution bit for bit (TMA path
    for W % 4 == 0 and r == 2, the simple kernel otherwise) and the oracle."""
    H, Wd = shape
    img = synth.uniform_f32(H * Wd, 700 + H, -1, 1).reshape(H, Wd)
    f = synth.uniform_f32((2 * r + 1) ** 2, 701, -1, 1).reshape(2 * r + 1, 2 * r + 1)
    for flags in (0, J.JACC_GRAPH_P2P):   # the local kernel; the peer push + finish kernels at world 1
        g, _ = make_graph(0, flags=flags)
        ext, out = _conv_band_graph(g, img, f, H, Wd, r)
        for _ in range(3):                 # three epochs: both staging parities of the peer path
            ext[:] = np.nan
            g.run()
            assert np.array_equal(ext, oracle.halo_band(img, 0, H, r)), flags
        g.destroy()
    plain = np.zeros_like(img)
    g, _ = make_graph(0)
    g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img, R), g.a(f, R), g.a(plain, W)], jacc.jacc_conv2d_params_t(H, Wd, r, 0))
    g.run()
    g.destroy()
    assert np.array_equal(out, plain)
    ref, ab = oracle.conv2d(img, f)
    assert np.all(np.abs(out.astype(np.float64) - ref) <= 1e-5 * ab + 1e-30)
