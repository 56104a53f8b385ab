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

// Row-block streaming ("CSR-stream"), for short rows: a block takes
// kRowsPerBlock consecutive rows, walks their contiguous non-zeros
// (row_ptr[r0] .. row_ptr[r1]) with coalesced loads of col / val, gathers x
// for every non-zero independently and leaves the products in shared memory;
// then thread i sums row r0 + i's products in k order.  A block whose rows
// hold more than kNnzCap non-zeros sums them row by row from global memory.
constexpr int kRowsPerBlock = 128, kNnzCap = 4096, kStreamThreads = 256;

template <int kB>   // non-zeros per thread per pass, their loads issued together
__global__ void __launch_bounds__(kStreamThreads) spmv_stream_kernel(const int32_t *__restrict__ row_ptr,
                                                                     const int32_t *__restrict__ col,
                                                                     const float *__restrict__ val,
                                                                     const float *__restrict__ x, float *__restrict__ y,
                                                                     int64_t n) {
    __shared__ float prod[kNnzCap];
    __shared__ int32_t rp[kRowsPerBlock + 1];
    const int64_t r0 = (int64_t)blockIdx.x * kRowsPerBlock;
    const int nr = (int)min((int64_t)kRowsPerBlock, n - r0);
    for (int i = threadIdx.x; i <= nr; i += kStreamThreads) rp[i] = __ldg(row_ptr + r0 + i);
    __syncthreads();
    const int32_t k0 = rp[0], cnt = rp[nr] - k0;
    if (cnt > kNnzCap) {   // long rows: one thread per row, straight from global memory
        for (int i = threadIdx.x; i < nr; i += kStreamThreads) {
            float acc = 0.f;
            for (int32_t k = rp[i]; k < rp[i + 1]; ++k) acc += __ldg(val + k) * __ldg(x + __ldg(col + k));
            y[r0 + i] = acc;
        }
        return;
    }
    // products, kB per thread per pass
    for (int base = threadIdx.x; base < cnt; base += kB * kStreamThreads) {
        int32_t c[kB];
        float v[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int k = base + u * kStreamThreads;
            c[u] = k < cnt ? ld_stream_i32(col + k0 + k) : 0;
            v[u] = k < cnt ? ld_stream_f32(val + k0 + k) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
            const int k = base + u * kStreamThreads;
            const float xv = __ldg(x + c[u]);
            if (k < cnt) prod[k] = v[u] * xv;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr; i += kStreamThreads) {
        float acc = 0.f;
        for (int k = rp[i] - k0; k < rp[i + 1] - k0; ++k) acc += prod[k];
        y[r0 + i] = acc;
    }
}

}  // namespace

cudaError_t spmv_csr_f32(const int32_t *row_ptr, const int32_t *col, const float *val, const float *x, float *y,
                         int64_t n, int64_t nnz, cudaStream_t st, int *launches) {
    if (n <= 0) return cudaSuccess;
    // Streaming row blocks for large matrices with short rows; the lane kernel
    // for L2-resident ones (measured, ms: 2M rows x 23 -- lane 0.134, stream
    // 128 rows / 4 loads 0.118, 64 rows 0.121, 256 rows 0.32, 8 loads 0.129;
    // 44609 rows -- lane 0.0122, stream 0.0135) and for long rows.  The
    // stream kernel is L1-bound on the x gathers (ncu L1TEX 88.6 %); 16-byte
    // col/val loads (0.118) and an x window staged in shared memory per block
    // (0.138-0.16) did not help
    if (n >= (1 << 18) && nnz <= (int64_t)n * (kNnzCap / kRowsPerBlock))
        spmv_stream_kernel<4><<<(unsigned)((n + kRowsPerBlock - 1) / kRowsPerBlock),
                                                         kStreamThreads, 0, st>>>(row_ptr, col, val, x, y, n);
    else
        spmv_kernel<kLanes, kBatch><<<(unsigned)((n * kLanes + 255) / 256), 256, 0, st>>>(row_ptr, col, val, x, y, n);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
