# compute-sanitizer (memcheck / racecheck / synccheck) over small graphs of every op
set -x
cat > /tmp/san.py <<'PY'
import numpy as np, sys
sys.path.insert(0, ".")
import synth
import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
R, W, RW = 1, 2, 3
g = J.Graph()
n = 20011
a, b = synth.vadd_inputs(n); c = np.zeros(n, np.float32); s = np.zeros(1, np.float32)
keys = synth.hist_keys(n + 3); bins = np.zeros(256, np.int32); big = np.zeros(1000, np.int32)
u = synth.bs_rand(n); call = np.zeros(n, np.float32); put = np.zeros(n, np.float32)
A, B = synth.sgemm_inputs(200, 300, 100, "signed"); C = np.zeros((200, 300), np.float32)
pos, vel = synth.nbody_state(700); pos2 = np.zeros_like(pos)
img = synth.uniform_f32(100 * 77, 1).reshape(100, 77); f = synth.uniform_f32(25, 2).reshape(5, 5); out = np.zeros_like(img)
bits = synth.corr_bitsets(70, 320); cc = np.zeros((70, 70), np.int32)
rp, col, val = synth.banded_csr(500, 5000, 30); x = synth.uniform_f32(500, 3); y = np.zeros(500, np.float32)
g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(bins, W)], jacc.jacc_hist_params_t(256))
g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(big, W)], jacc.jacc_hist_params_t(1000))
g.add_task(J.JACC_OP_BLACKSCHOLES_F32, [g.a(u, R), g.a(call, W), g.a(put, W)])
g.add_task(J.JACC_OP_SGEMM_F32, [g.a(A, R), g.a(B, R), g.a(C, W)], jacc.jacc_sgemm_params_t(200, 300, 100, 100, 300, 300, 0, 0))
g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(pos, R, f32x4=True), g.a(vel, RW, f32x4=True), g.a(pos2, W, f32x4=True)], jacc.jacc_nbody_params_t(0, 0.016, 0.01, 1.0))
g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img, R), g.a(f, R), g.a(out, W)], jacc.jacc_conv2d_params_t(100, 77, 2, 0))
g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(bits.view(np.int32), R), g.a(bits.view(np.int32), R), g.a(cc, W)], jacc.jacc_corr_params_t(70, 70, 10))
g.add_task(J.JACC_OP_SPMV_CSR_F32, [g.a(rp, R), g.a(col, R), g.a(val, R), g.a(x, R), g.a(y, W)], jacc.jacc_spmv_params_t(500, 500))
# paths added later in round 1: conv2d TMA kernel (W % 4 == 0, radius 2), corr and
# SGEMM split-K, N-body mixed grid (a 2^14-target shard of 2^16 sources: 1376 3-pair units)
img2 = synth.uniform_f32(67 * 132, 4).reshape(67, 132); out2 = np.zeros_like(img2)
img3 = synth.uniform_f32(4736 * 4096, 6).reshape(4736, 4096); out3 = np.zeros_like(img3)   # the 128-wide-tile TMA config (2368 tiles)
bits2 = synth.corr_bitsets(100, 16384); cc2 = np.zeros((100, 100), np.int32)
A2, B2 = synth.sgemm_inputs(300, 520, 1000, "signed"); C2 = np.zeros((300, 520), np.float32)
pos3, vel3 = synth.nbody_state(1 << 16); vel3 = vel3[:1 << 14].copy(); pos4 = np.zeros_like(vel3)
g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img2, R), g.a(f, R), g.a(out2, W)], jacc.jacc_conv2d_params_t(67, 132, 2, 0))
g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(bits2.view(np.int32), R), g.a(bits2.view(np.int32), R), g.a(cc2, W)], jacc.jacc_corr_params_t(100, 100, 512))
g.add_task(J.JACC_OP_SGEMM_F32, [g.a(A2, R), g.a(B2, R), g.a(C2, W)], jacc.jacc_sgemm_params_t(300, 520, 1000, 1000, 520, 520, 0, 0))
g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(pos3, R, f32x4=True), g.a(vel3, RW, f32x4=True), g.a(pos4, W, f32x4=True)], jacc.jacc_nbody_params_t(1 << 14, 0.016, 0.01, 1.0))
g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img3, R), g.a(f, R), g.a(out3, W)], jacc.jacc_conv2d_params_t(4736, 4096, 2, 0))
# round 2: the pre-split SGEMM fallback (K = 101: lda not a multiple of 4; the
# default 16-byte-aligned shapes above take the CTA-pair kernel), the halo
# exchange + halo-row convolution (TMA and simple kernels), an RW histogram
A3, B3 = synth.sgemm_inputs(130, 260, 101, "signed"); C3 = np.zeros((130, 260), np.float32)
g.add_task(J.JACC_OP_SGEMM_F32, [g.a(A3, R), g.a(B3, R), g.a(C3, W)], jacc.jacc_sgemm_params_t(130, 260, 101, 101, 260, 260, 0, 0))
for (hh, ww) in ((70, 132), (45, 77)):
    band = synth.uniform_f32(hh * ww, 7).reshape(hh, ww); ext = np.zeros((hh + 4, ww), np.float32); ob = np.zeros_like(band)
    g.add_task(J.JACC_OP_HALO_EXCHANGE_F32, [g.a(band, R), g.a(ext, W)], jacc.jacc_halo_params_t(hh, ww, 2, 0))
    g.add_task(J.JACC_OP_CONV2D_F32, [g.a(ext, R), g.a(f, R), g.a(ob, W)], jacc.jacc_conv2d_params_t(hh, ww, 2, J.JACC_CONV2D_HALO_ROWS))
bins_rw = np.ones(256, np.int32)
g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(bins_rw, RW)], jacc.jacc_hist_params_t(256))
# round 2 (later): the 256-bit vadd (>= 2^26 elements, ragged tail), Black-Scholes
# through its 256-bit (graph copies) and 128-bit (16-byte aligned view) kernels,
# corr with 16-bit split partials (bits2 above) and 32-bit ones (2^20 documents)
import torch
nv = (1 << 26) + 5
va = torch.rand(nv, device="cuda"); vb = torch.rand(nv, device="cuda"); vc = torch.empty(nv, device="cuda")
g.add_task(J.JACC_OP_VADD_F32, [g.a(va, R), g.a(vb, R), g.a(vc, W)])
ub = torch.rand(n + 8, device="cuda"); cb = torch.zeros(n + 8, device="cuda"); pb = torch.zeros(n + 8, device="cuda")
g.add_task(J.JACC_OP_BLACKSCHOLES_F32, [g.a(ub[4:4 + n], R), g.a(cb[4:4 + n], W), g.a(pb[4:4 + n], W)])
bits3 = synth.corr_bitsets(100, 1 << 20); cc3 = np.zeros((100, 100), np.int32)
g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(bits3.view(np.int32), R), g.a(bits3.view(np.int32), R), g.a(cc3, W)], jacc.jacc_corr_params_t(100, 100, 1 << 15))
bits4 = synth.corr_bitsets(1536, 4096); cc4 = np.zeros((1536, 1536), np.int32)   # the CTA-pair corr kernel, (2, 1, 2) clusters
g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(bits4.view(np.int32), R), g.a(bits4.view(np.int32), R), g.a(cc4, W)], jacc.jacc_corr_params_t(1536, 1536, 128))
g.run(); g.run()
print("ok", g.stats()["launches"])
g.destroy()
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san.py > gpurun_out/san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -3 gpurun_out/san_$tool.txt
done
