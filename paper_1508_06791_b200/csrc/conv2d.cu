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
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {

constexpr int TX = 32, TY = 32, Q = 4;     // tile, outputs per thread (rows)

template <int R>
__global__ void __launch_bounds__(256) conv2d_kernel(const float *__restrict__ img, int64_t H, int64_t W,
                                                     const float *__restrict__ filt, float *__restrict__ out) {
    constexpr int K = 2 * R + 1, SW = TX + 2 * R, SH = TY + 2 * R;
    __shared__ float s[SH][SW + 1];
    __shared__ float fs[K * K];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
    const int64_t x0 = (int64_t)blockIdx.x * TX, y0 = (int64_t)blockIdx.y * TY;
    if (threadIdx.x < K * K) fs[threadIdx.x] = filt[threadIdx.x];
    for (int idx = threadIdx.x; idx < SH * SW; idx += 256) {
        const int sy = idx / SW, sx = idx - sy * SW;
        const int64_t gy = y0 - R + sy, gx = x0 - R + sx;
        s[sy][sx] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? __ldg(img + gy * W + gx) : 0.f;
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

}  // namespace

cudaError_t conv2d_f32(const float *img, int64_t H, int64_t W, const float *filt, int radius, float *out,
                       cudaStream_t st, int *launches) {
    if (H <= 0 || W <= 0) return cudaSuccess;
    dim3 grid((unsigned)((W + TX - 1) / TX), (unsigned)((H + TY - 1) / TY));
    switch (radius) {
        case 1: conv2d_kernel<1><<<grid, 256, 0, st>>>(img, H, W, filt, out); break;
        case 2: conv2d_kernel<2><<<grid, 256, 0, st>>>(img, H, W, filt, out); break;
        case 3: conv2d_kernel<3><<<grid, 256, 0, st>>>(img, H, W, filt, out); break;
        case 4: conv2d_kernel<4><<<grid, 256, 0, st>>>(img, H, W, filt, out); break;
        default: return cudaErrorInvalidValue;
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
