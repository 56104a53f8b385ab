// spmv.cu -- Sparse matrix-vector multiply, CSR (PAPER.md
// §4.2: bcsstk32, 44609 x 44609, 1029655 non-zeros; "irregular memory
// access ... does not favor GPGPU execution").  Reading R22:
//   y[i] = sum_{k = row_ptr[i]}^{row_ptr[i+1]-1} val[k] x[col[k]]
// Gather-bound: 8 algorithmic bytes per non-zero (val + col) plus the row
// pointers and y; x is gathered through the read-only path (mostly L1/L2
// hits for a banded matrix).  ~23 non-zeros per row, so 8 lanes share a row
// (4 rows per warp): coalesced val/col streams, shuffle-xor reduction.
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {

constexpr int kLanesPerRow = 8;

__global__ void __launch_bounds__(256) spmv_kernel(const int32_t *__restrict__ row_ptr,
                                                   const int32_t *__restrict__ col, const float *__restrict__ val,
                                                   const float *__restrict__ x, float *__restrict__ y, int64_t n) {
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = gt / kLanesPerRow;
    const int sub = threadIdx.x & (kLanesPerRow - 1);
    float acc = 0.f;
    if (row < n) {
        const int32_t k0 = __ldg(row_ptr + row), k1 = __ldg(row_ptr + row + 1);
        for (int32_t k = k0 + sub; k < k1; k += kLanesPerRow) acc = fmaf(__ldg(val + k), __ldg(x + __ldg(col + k)), acc);
    }
#pragma unroll
    for (int o = kLanesPerRow / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (row < n && sub == 0) y[row] = acc;
}

}  // namespace

cudaError_t spmv_csr_f32(const int32_t *row_ptr, const int32_t *col, const float *val, const float *x, float *y,
                         int64_t n, cudaStream_t st, int *launches) {
    if (n <= 0) return cudaSuccess;
    const int64_t threads = n * kLanesPerRow;
    spmv_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(row_ptr, col, val, x, y, n);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
