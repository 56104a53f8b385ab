// conv2d.cu -- 2D convolution (§4.2, P:489-490:
// "convolves a 2048 x 2048 image with a 5 x 5 filter").  Reading R20: true
// convolution (filter flipped), zero padding, same-size output:
//   out[y][x] = sum_{i,j=0}^{2r} f[i][j] img[y + r - i][x + r - j]
//
// sm_100a design: a stencil map, HBM-bound at 8 algorithmic bytes per pixel
// (read the image once, write the output once) when the tile reuse stays on
// chip.  32 x 32 output tile per 256-thread block; the (32 + 2r)^2 input tile
// (halo zero-filled at the image border) is staged once in shared memory;
// the (2r+1)^2 filter lives in registers; each thread produces a column of 4
// outputs and slides a (4 + 2r)-tall register window over the tile, so every
// shared-memory value it loads feeds up to (2r+1) FMAs.
//
// TMA path (row stride a multiple of 16 bytes, radius 2 = the paper's 5 x 5):
// persistent blocks walk PX x 64 output tiles in row-major order (PX = 128
// for large images, 64 when there are few tiles); the (PX + 8) x (64 + 2r)
// input box of each tile (x from x0 - 4, y from y0 - r) arrives by one
// cp.async.bulk.tensor 2-D load into an mbarrier ring, and TMA's
// out-of-bounds zero fill IS the zero padding on all four sides.  The box
// starts 4 columns (16 bytes) left of the tile because the innermost start
// coordinate must be a multiple of 16 bytes -- measured on the box with
// scripts/micro/tma_probe.cu: x = -2 or 250 (floats) faults with an illegal
// instruction, x = -4 / 252 and any row coordinate work, out-of-range parts
// zero-filled.  Each thread computes two x-adjacent outputs over QR rows with
// the paired FP32 instruction FFMA2 (input value broadcast, a pair of filter
// weights), sliding down its (2 + 2r)-wide window with 8-byte shared loads so
// every loaded row feeds up to 2r + 1 output rows; outputs leave as 8-byte
// streaming stores.  Other shapes use the simple kernel below.
#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace jacc_k {
namespace {

constexpr int TX = 32, TY = 32, Q = 4;     // tile, outputs per thread (rows)

// TMA path configurations: output tile PX x 64, QR output rows per thread
// (x 2 columns, 256 threads), ring depth.  Measured at 16384^2 (ms, same-box
// A/B): 64 x 64 / QR 8 / 3 stages 0.387, 4 stages 0.388; 128 x 64 / QR 16 /
// 2 stages 0.367, 3 stages 0.396.  At 2048^2 (512 tiles, L2-resident) the
// 64-wide tile is faster (16.9 vs 18.7 us): more tiles than blocks.
template <int PX_, int QR_, int kStages_>
struct TmaCfg {
    static constexpr int PX = PX_, PY = 64, QR = QR_, kStages = kStages_;
    static_assert((PX / 2) * (PY / QR) == 256, "256 threads: PX / 2 column pairs x PY / QR row groups");
};
using CfgSmall = TmaCfg<64, 8, 3>;
using CfgLarge = TmaCfg<128, 16, 2>;

template <int R, class C>
struct Box {
    static constexpr int X0 = 4;                      // box starts 4 floats (16 B) left of the tile
    static constexpr int W = C::PX + 2 * X0;          // covers x0 - 4 .. x0 + PX + 3
    static constexpr int H = C::PY + 2 * R;
    static constexpr int kBytes = W * H * 4;
    static constexpr int kStride = (kBytes + 1023) & ~1023;   // TMA destinations: 128-byte (here 1 KiB) aligned
    static constexpr int kSmem = C::kStages * kStride + 1024; // + alignment slack of the dynamic base
    static_assert(R <= X0 && ((X0 - R) & 1) == 0, "window start must be even (8-byte shared loads)");
};

__device__ __forceinline__ void st_stream2(float *p, float2 v) {
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}

template <int R, class C>
__global__ void __launch_bounds__(256, 2) conv2d_tma_kernel(const __grid_constant__ CUtensorMap map, int64_t H,
                                                            int64_t W, const float *__restrict__ filt,
                                                            float *__restrict__ out, int tiles_x, int ntiles,
                                                            int y_off) {
    constexpr int K = 2 * R + 1, BW = Box<R, C>::W, PX = C::PX, PY = C::PY, QR = C::QR, kStages = C::kStages;
    constexpr uint32_t kBytes = Box<R, C>::kBytes;
    constexpr int kStrideF = Box<R, C>::kStride / 4;         // floats between ring stages
    extern __shared__ uint8_t smem_raw[];
    // kStages boxes, 1 KiB aligned; offset arithmetic on the shared array (not
    // through an integer) keeps the loads below LDS instead of generic LD
    float *ring = reinterpret_cast<float *>(smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u));
    __shared__ __align__(8) uint64_t bar[kStages];
    const int tid = threadIdx.x, cx = tid % (PX / 2), rg = tid / (PX / 2);   // column pair, row group (QR rows)
    // Weights of the thread's input column j (j = 0 .. K) in its output pair
    // (c, c + 1): lo takes w(m, j), hi takes w(m, j - 1), w = the flipped
    // filter.  Inner columns are one FFMA2 with the input value broadcast to
    // both halves (no re-pairing of adjacent inputs into operand pairs: that
    // cost ~8 MOVs per output), the outer two a plain FFMA on one half.  The
    // (w(m, j), w(m, j - 1)) pairs are built in shared memory and loaded as
    // pairs, so the compiler keeps 20 pair registers instead of re-pairing 25
    // scalars with MOVs.  Per output: 10 FFMA2 + 5 FFMA, summed in the same
    // order as the oracle's definition (filter column by filter column).
    __shared__ float2 gtab[K * (K - 1)];
    if (tid < K * (K - 1)) {
        const int m = tid / (K - 1), j = tid % (K - 1) + 1;
        gtab[tid] = make_float2(__ldg(filt + (2 * R - m) * K + (2 * R - j)),
                                __ldg(filt + (2 * R - m) * K + (2 * R - j + 1)));
    }
    // (the map's address is taken directly in the kernel body: through a
    // capturing lambda nvcc 12.9 passed the wrong parameter slot to UTMALDG)
#define CONV_ISSUE(t_, stage_)                                                                     \
    do {                                                                                           \
        const int x0_ = ((t_) % tiles_x) * PX, y0_ = ((t_) / tiles_x) * PY;                       \
        const uint32_t b_ = tc::smem_u32(&bar[(stage_)]);                                          \
        tc::mbar_expect_tx(b_, kBytes);                                                            \
        tc::tma_load_2d(tc::smem_u32(ring + (stage_) * kStrideF), &map, x0_ - Box<R, C>::X0, y0_ + y_off - R, b_); \
    } while (0)
    if (tid == 0) {
        tc::tma_prefetch(&map);
        for (int i = 0; i < kStages; ++i) tc::mbar_init(tc::smem_u32(&bar[i]), 1);
        tc::fence_barrier_init();
        for (int i = 0; i < kStages - 1; ++i)
            if (blockIdx.x + i * (int)gridDim.x < ntiles) CONV_ISSUE(blockIdx.x + i * (int)gridDim.x, i);
    }
    __syncthreads();
    float2 gp[K * (K - 1)];
#pragma unroll
    for (int i = 0; i < K * (K - 1); ++i) gp[i] = gtab[i];
    // tile coordinates advanced incrementally (no division per tile)
    const int dtx = (int)gridDim.x % tiles_x, dty = (int)gridDim.x / tiles_x;
    int tx = blockIdx.x % tiles_x, ty = blockIdx.x / tiles_x;
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int stage = k % kStages;
        const int tn = t + (kStages - 1) * gridDim.x;   // refill the stage freed in iteration k - 1
        if (tid == 0 && tn < ntiles) CONV_ISSUE(tn, (k + kStages - 1) % kStages);
        tc::mbar_wait(tc::smem_u32(&bar[stage]), (k / kStages) & 1);
        const float *S = ring + stage * kStrideF + (rg * QR) * BW + 2 * cx + (Box<R, C>::X0 - R);
        float2 acc[QR];
#pragma unroll
        for (int q = 0; q < QR; ++q) acc[q] = make_float2(0.f, 0.f);
#pragma unroll
        for (int w = 0; w < QR + 2 * R; ++w) {   // window row w feeds output rows q = w - m
            float v[2 + 2 * R];
#pragma unroll
            for (int c = 0; c <= R; ++c) {
                const float2 p = *reinterpret_cast<const float2 *>(S + w * BW + 2 * c);
                v[2 * c] = p.x;
                v[2 * c + 1] = p.y;
            }
#pragma unroll
            for (int q = 0; q < QR; ++q) {
                const int m = w - q;
                if (m < 0 || m > 2 * R) continue;
#pragma unroll
                acc[q].x = fmaf(gp[m * (K - 1)].y, v[0], acc[q].x);
#pragma unroll
                for (int j = 1; j < K; ++j)
                    acc[q] = __ffma2_rn(gp[m * (K - 1) + j - 1], make_float2(v[j], v[j]), acc[q]);
                acc[q].y = fmaf(gp[m * (K - 1) + K - 2].x, v[K], acc[q].y);
            }
        }
        const int64_t xo = (int64_t)tx * PX + 2 * cx, yo = (int64_t)ty * PY + rg * QR;
        if (xo < W) {
#pragma unroll
            for (int q = 0; q < QR; ++q)
                if (yo + q < H) st_stream2(out + (yo + q) * W + xo, acc[q]);
        }
        tx += dtx;
        ty += dty;
        if (tx >= tiles_x) {
            tx -= tiles_x;
            ++ty;
        }
        __syncthreads();   // every thread is done with `stage` before it is refilled
    }
#undef CONV_ISSUE
}

template <int R>
__global__ void __launch_bounds__(256) conv2d_kernel(const float *__restrict__ img, int64_t H_in, int64_t W,
                                                     const float *__restrict__ filt, float *__restrict__ out,
                                                     int64_t y_off, int64_t H) {
    constexpr int K = 2 * R + 1, SW = TX + 2 * R, SH = TY + 2 * R;
    __shared__ float s[SH][SW + 1];
    __shared__ float fs[K * K];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const int64_t x0 = (int64_t)blockIdx.x * TX, y0 = (int64_t)blockIdx.y * TY;
    if (threadIdx.x < K * K) fs[threadIdx.x] = filt[threadIdx.x];
    for (int idx = threadIdx.x; idx < SH * SW; idx += 256) {
        const int sy = idx / SW, sx = idx - sy * SW;
        const int64_t gy = y0 + y_off - R + sy, gx = x0 - R + sx;
        s[sy][sx] = (gy >= 0 && gy < H_in && gx >= 0 && gx < W) ? __ldg(img + gy * W + gx) : 0.f;
    }
    __syncthreads();
    float f[K * K];
#pragma unroll
    for (int i = 0; i < K * K; ++i) f[i] = fs[i];
    float acc[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) acc[q] = 0.f;
    const int ly0 = ty * Q;
#pragma unroll
    for (int c = 0; c <= 2 * R; ++c) {          // column offset = 2R - j
        float v[Q + 2 * R];
#pragma unroll
        for (int m = 0; m < Q + 2 * R; ++m) v[m] = s[ly0 + m][tx + c];
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
            for (int i = 0; i < K; ++i) acc[q] = fmaf(f[i * K + (2 * R - c)], v[q + 2 * R - i], acc[q]);
    }
    const int64_t x = x0 + tx;
    if (x < W) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int64_t y = y0 + ly0 + q;
            if (y < H) out[y * W + x] = acc[q];
        }
    }
}

template <int R, class C>
cudaError_t launch_tma_cfg(const float *img, int64_t H_in, int64_t W, const float *filt, float *out,
                           int64_t y_off, int64_t H, cudaStream_t st, bool *done) {
    *done = false;
    CUtensorMap map;
    if (!tc::make_map_2d(&map, img, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, H_in, W, W * 4, Box<R, C>::H, Box<R, C>::W,
                         0))
        return cudaSuccess;   // no tensor map for this shape: the simple kernel runs
    const int smem = Box<R, C>::kSmem;
    cudaError_t e = set_max_dyn_smem((const void *)conv2d_tma_kernel<R, C>, smem);
    if (e != cudaSuccess) return e;
    const int64_t tiles_x = (W + C::PX - 1) / C::PX, ntiles = tiles_x * ((H + C::PY - 1) / C::PY);
    int64_t grid = (int64_t)sm_count() * blocks_per_sm((const void *)conv2d_tma_kernel<R, C>, 256, smem);
    if (grid > ntiles) grid = ntiles;
    conv2d_tma_kernel<R, C><<<(unsigned)grid, 256, smem, st>>>(map, H, W, filt, out, (int)tiles_x, (int)ntiles,
                                                               (int)y_off);
    *done = true;
    return cudaGetLastError();
}

template <int R>
cudaError_t launch_tma(const float *img, int64_t H_in, int64_t W, const float *filt, float *out, int64_t y_off,
                       int64_t H, cudaStream_t st, bool *done) {
    // the wide tile once there are >= 16 of its tiles per SM (HBM-streaming sizes)
    const int64_t wide_tiles = ((W + CfgLarge::PX - 1) / CfgLarge::PX) * ((H + CfgLarge::PY - 1) / CfgLarge::PY);
    if (wide_tiles >= 16 * (int64_t)sm_count())
        return launch_tma_cfg<R, CfgLarge>(img, H_in, W, filt, out, y_off, H, st, done);
    return launch_tma_cfg<R, CfgSmall>(img, H_in, W, filt, out, y_off, H, st, done);
}

}  // namespace

// Output rows [y_off, y_off + H) of the convolution of the H_in-row image
// (zero padded outside it), written to out rows [0, H): y_off = 0, H = H_in
// is the plain same-size convolution; y_off = r, H_in = H + 2r convolves a
// row band that carries its r halo rows above and below
// (JACC_CONV2D_HALO_ROWS), so no output row touches the padding in y.
cudaError_t conv2d_f32(const float *img, int64_t H_in, int64_t W, const float *filt, int radius, float *out,
                       int64_t y_off, int64_t H, cudaStream_t st, int *launches) {
    if (H <= 0 || W <= 0) return cudaSuccess;
    // TMA path: 16-byte aligned rows, 8-byte aligned output (its v2 stores),
    // int32 tile coordinates
    if (radius == 2 && W % 4 == 0 && aligned16(img) && ((uintptr_t)out & 7) == 0 && (W + 128) < (1ll << 31) &&
        (H_in + 64) < (1ll << 31) && ((W + 63) / 64) * ((H + 63) / 64) < (1ll << 31)) {
        bool done = false;
        cudaError_t e = launch_tma<2>(img, H_in, W, filt, out, y_off, H, st, &done);
        if (e != cudaSuccess) return e;
        if (done) {
            ++*launches;
            return cudaSuccess;
        }
    }
    dim3 grid((unsigned)((W + TX - 1) / TX), (unsigned)((H + TY - 1) / TY));
    switch (radius) {
        case 1: conv2d_kernel<1><<<grid, 256, 0, st>>>(img, H_in, W, filt, out, y_off, H); break;
        case 2: conv2d_kernel<2><<<grid, 256, 0, st>>>(img, H_in, W, filt, out, y_off, H); break;
        case 3: conv2d_kernel<3><<<grid, 256, 0, st>>>(img, H_in, W, filt, out, y_off, H); break;
        case 4: conv2d_kernel<4><<<grid, 256, 0, st>>>(img, H_in, W, filt, out, y_off, H); break;
        default: return cudaErrorInvalidValue;
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
