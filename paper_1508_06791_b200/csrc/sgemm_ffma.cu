// sgemm_ffma.cu -- Dense matrix multiply (§4.2, P:484-485, P:525:
// SGEMM), C = A.B row-major, beta = 0 (reading R13), JACC_SGEMM_FFMA mode:
// a plain fp32 SIMT kernel -- 128x128 block tile, BK = 8, 256 threads with
// an 8x8 register micro-tile each, shared-memory staging with zero-filled
// edges.  This is the parity baseline the tcgen05 3xTF32 path
// (sgemm_tcgen05.cu) is measured against; it never runs unless asked for.
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {

namespace {
constexpr int BM = 128, BN = 128, BK = 8, TM = 8, TN = 8;

__global__ void __launch_bounds__(256) sgemm_ffma_kernel(const float *__restrict__ A, const float *__restrict__ B,
                                                         float *__restrict__ C, int64_t M, int64_t N, int64_t K,
                                                         int64_t lda, int64_t ldb, int64_t ldc) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int ty = tid / 16, tx = tid % 16;
    const int64_t row0 = (int64_t)blockIdx.y * BM, col0 = (int64_t)blockIdx.x * BN;
    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;
    const int ar = tid / 2, ac = (tid % 2) * 4;    // A tile 128 x 8
    const int br = tid / 32, bc = (tid % 32) * 4;  // B tile 8 x 128
    for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t r = row0 + ar, c = k0 + ac + q;
            As[ac + q][ar] = (r < M && c < K) ? A[r * lda + c] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int64_t r = k0 + br, c = col0 + bc + q;
            Bs[br][bc + q] = (r < K && c < N) ? B[r * ldb + c] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = As[kk][ty * TM + i];
#pragma unroll
            for (int j = 0; j < TN; ++j) b[j] = Bs[kk][tx * TN + j];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int64_t r = row0 + ty * TM + i;
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int64_t c = col0 + tx * TN + j;
            if (c < N) C[r * ldc + c] = acc[i][j];
        }
    }
}
}  // namespace

cudaError_t sgemm_ffma(const float *A, const float *B, float *C, const jacc_sgemm_params_t *p, cudaStream_t st,
                       int *launches) {
    if (p->M == 0 || p->N == 0) return cudaSuccess;
    dim3 grid((unsigned)((p->N + BN - 1) / BN), (unsigned)((p->M + BM - 1) / BM));
    sgemm_ffma_kernel<<<grid, 256, 0, st>>>(A, B, C, p->M, p->N, p->K, p->lda, p->ldb, p->ldc);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
