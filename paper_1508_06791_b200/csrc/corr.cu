// corr.cu -- Correlation matrix (§4.2: the
// Lucene OpenBitSet "intersection count", 1024 terms x 16384 documents;
// Jacc wins by using the GPU's `popc`).  Reading R21:
//   C[i][j] = sum_w popcount(A_i[w] & B_j[w])     (term bitsets, 32-bit words)
// Integer, bit-exact.  A binary "GEMM": 64 x 64 output tile per 256-thread
// block, 32-word K slices of both bitset tiles staged in shared memory
// (word-major, padded), 4 x 4 counts per thread in registers, one LOP3 AND +
// POPC + IADD per bit-word pair.  tcgen05 has no 1-bit kind, so this runs on
// the integer pipes.
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {

constexpr int BT = 64, BW = 32;

__global__ void __launch_bounds__(256) corr_kernel(const uint32_t *__restrict__ A, int64_t ta,
                                                   const uint32_t *__restrict__ B, int64_t tb, int64_t words,
                                                   int32_t *__restrict__ C) {
    __shared__ uint32_t As[BW][BT + 1];
    __shared__ uint32_t Bs[BW][BT + 1];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t i0 = (int64_t)blockIdx.y * BT, j0 = (int64_t)blockIdx.x * BT;
    int32_t acc[4][4] = {};
    for (int64_t w0 = 0; w0 < words; w0 += BW) {
        // 64 rows x 32 words per operand: thread loads rows r = tid/32 + 8q, word tid%32
#pragma unroll
        for (int q = 0; q < BT / 8; ++q) {
            const int r = (tid >> 5) + 8 * q, w = tid & 31;
            const int64_t gi = i0 + r, gj = j0 + r, gw = w0 + w;
            As[w][r] = (gi < ta && gw < words) ? __ldg(A + gi * words + gw) : 0u;
            Bs[w][r] = (gj < tb && gw < words) ? __ldg(B + gj * words + gw) : 0u;
        }
        __syncthreads();
#pragma unroll 8
        for (int w = 0; w < BW; ++w) {
            uint32_t a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) { a[u] = As[w][ty * 4 + u]; b[u] = Bs[w][tx * 4 + u]; }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] += __popc(a[u] & b[v]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t i = i0 + ty * 4 + u;
        if (i >= ta) continue;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int64_t j = j0 + tx * 4 + v;
            if (j < tb) C[i * tb + j] = acc[u][v];
        }
    }
}

}  // namespace

cudaError_t corr_popc_u32(const uint32_t *A, int64_t ta, const uint32_t *B, int64_t tb, int64_t words, int32_t *C,
                          cudaStream_t st, int *launches) {
    if (ta <= 0 || tb <= 0) return cudaSuccess;
    dim3 grid((unsigned)((tb + BT - 1) / BT), (unsigned)((ta + BT - 1) / BT));
    corr_kernel<<<grid, 256, 0, st>>>(A, ta, B, tb, words, C);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
