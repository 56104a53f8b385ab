// spmv.cu -- Sparse matrix-vector multiply, CSR (PAPER.md
// §4.2: bcsstk32, 44609 x 44609, 1029655 non-zeros; "irregular memory
// access ... does not favor GPGPU execution").  Reading R22:
//   y[i] = sum_{k = row_ptr[i]}^{row_ptr[i+1]-1} val[k] x[col[k]]
// Gather-bound: 8 algorithmic bytes per non-zero (val + col) plus the row
// pointers and y; x is gathered through the read-only path (mostly L1/L2
// hits for a banded matrix).  ~23 non-zeros per row: 4 lanes share a row
// (8 rows per warp), each lane loading its ~6 column indices and values
// first and then gathering x for all of them, so each row costs two
// dependent memory round trips, not two per non-zero; shuffle-xor reduction.
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {


__device__ __forceinline__ int32_t ld_stream_i32(const int32_t *p) {
    int32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ float ld_stream_f32(const float *p) {
    float r;
    asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}

// Measured at 4M rows x 23 non-zeros (ms): 8 lanes x 1 non-zero per pass
// (the first version) 0.36; 8 x 4 0.29; 16 x 2 0.47; 4 x 6 0.256; 4 x 8
// 0.256; 2 x 12 0.33; 1 x 24 0.57; two rows per thread 0.32.
constexpr int kLanes = 4, kBatch = 6;

template <int L, int B>   // L lanes per row, B non-zeros per lane per pass
__global__ void __launch_bounds__(256) spmv_kernel(const int32_t *__restrict__ row_ptr,
                                                   const int32_t *__restrict__ col, const float *__restrict__ val,
                                                   const float *__restrict__ x, float *__restrict__ y, int64_t n) {
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = gt / L;
    const int sub = threadIdx.x & (L - 1);
    float acc = 0.f;
    if (row < n) {
        const int32_t k0 = __ldg(row_ptr + row), k1 = __ldg(row_ptr + row + 1);
        // B non-zeros per lane per pass: every column index and value is
        // loaded first (streaming, read once), then the B x gathers are
        // independent -- 2 memory round trips per pass instead of 2 per
        // non-zero.  The lane still adds its products in k order.
        for (int32_t k = k0 + sub; k < k1; k += B * L) {
            int32_t c[B];
            float v[B];
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const int32_t kk = k + u * L;
                c[u] = kk < k1 ? ld_stream_i32(col + kk) : 0;
                v[u] = kk < k1 ? ld_stream_f32(val + kk) : 0.f;
            }
            float xv[B];
#pragma unroll
            for (int u = 0; u < B; ++u) xv[u] = __ldg(x + c[u]);
#pragma unroll
            for (int u = 0; u < B; ++u)
                if (k + u * L < k1) acc = fmaf(v[u], xv[u], acc);
        }
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (row < n && sub == 0) y[row] = acc;
}

}  // namespace

cudaError_t spmv_csr_f32(const int32_t *row_ptr, const int32_t *col, const float *val, const float *x, float *y,
                         int64_t n, cudaStream_t st, int *launches) {
    if (n <= 0) return cudaSuccess;
    spmv_kernel<kLanes, kBatch><<<(unsigned)((n * kLanes + 255) / 256), 256, 0, st>>>(row_ptr, col, val, x, y, n);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
