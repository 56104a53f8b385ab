// corr.cu -- Correlation matrix (§4.2: the
// Lucene OpenBitSet "intersection count", 1024 terms x 16384 documents;
// Jacc wins by using the GPU's `popc`).  Reading R21:
//   C[i][j] = sum_w popcount(A_i[w] & B_j[w])     (term bitsets, 32-bit words)
// Integer, bit-exact.
//
// The intersection count IS a dense contraction: with X[i][d] = bit d of term
// i (0/1), C = X_A . X_B^T.  On sm_100a that belongs on the 5th-generation
// tensor cores (tcgen05 has no 1-bit kind; the legacy mma.sync b1 path lowers
// to 8 IMMA.U8 per instruction), so:
//   1. unpack: bitsets -> 0/1 uint8 rows (K-major), zero padded to the tile grid;
//   2. GEMM: tcgen05.mma.cta_group::1.kind::i8 (u8 x u8 -> s32, exact),
//      128 x 64 output tile per CTA, 128-byte K blocks staged by TMA (128B
//      swizzle) through a 4-stage mbarrier ring, accumulator in TMEM (64
//      columns), epilogue tcgen05.ld -> int32 stores.
// One warp issues TMA, one thread issues the MMAs, four warps drain TMEM.
#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace jacc_k {
namespace {

constexpr int BM = 128, BN = 64, BK = 128;     // BK bytes = one 128 B swizzle row of u8
constexpr int kStages = 4;
constexpr int kABytes = BM * BK, kBBytes = BN * BK;
constexpr int kStageBytes = kABytes + kBBytes;  // 24 KB
constexpr int kThreads = 192;
constexpr int kTmemCols = 64;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
// kind::i8: D = s32 (c_format 2), A/B unsigned 8-bit (format 0), K-major, M = 128, N = 64
constexpr uint32_t kIdesc = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// bitsets [t x words] -> u8 [tp x kp]: byte d of row i = bit d%32 of word d/32
__global__ void __launch_bounds__(256) unpack_kernel(const uint32_t *__restrict__ bits, int64_t t, int64_t words,
                                                     uint8_t *__restrict__ x, int64_t tp, int64_t kp) {
    const int64_t wpr = kp / 32;   // 32 bytes (one word) per thread
    const int64_t total = tp * wpr;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = q / wpr, w = q - r * wpr;
        const uint32_t v = (r < t && w < words) ? __ldg(bits + r * words + w) : 0u;
        uint4 o[2];
        uint32_t *ob = (uint32_t *)o;
#pragma unroll
        for (int b = 0; b < 8; ++b) {   // 4 bits -> 4 bytes (little endian)
            const uint32_t nib = (v >> (4 * b)) & 0xFu;
            ob[b] = (nib & 1u) | ((nib >> 1) & 1u) << 8 | ((nib >> 2) & 1u) << 16 | ((nib >> 3) & 1u) << 24;
        }
        uint4 *dst = (uint4 *)(x + r * kp + w * 32);
        dst[0] = o[0];
        dst[1] = o[1];
    }
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accum));
}

__global__ void __launch_bounds__(kThreads, 1)
    corr_i8_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   int32_t *__restrict__ C, int64_t ta, int64_t tb, int num_kb) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *bars = (uint64_t *)(smem + kStages * kStageBytes);
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kStages + 1);
    const uint32_t full0 = tc::smem_u32(bars), empty0 = tc::smem_u32(bars + kStages),
                   tfull = tc::smem_u32(bars + 2 * kStages);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_blk = blockIdx.y, n_blk = blockIdx.x;
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&map_a);
        tc::tma_prefetch(&map_b);
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(full0 + 8 * s, 1);
            tc::mbar_init(empty0 + 8 * s, 1);
        }
        tc::mbar_init(tfull, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::alloc_cols(tc::smem_u32(tmem_slot), kTmemCols);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_d = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {   // TMA producer
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % kStages;
                tc::mbar_wait(empty0 + 8 * s, ((kb / kStages) & 1) ^ 1);
                uint8_t *st = smem + s * kStageBytes;
                tc::mbar_expect_tx(full0 + 8 * s, kStageBytes);
                tc::tma_load_2d(tc::smem_u32(st), &map_a, kb * BK, m_blk * BM, full0 + 8 * s);
                tc::tma_load_2d(tc::smem_u32(st + kABytes), &map_b, kb * BK, n_blk * BN, full0 + 8 * s);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // MMA issuer
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % kStages;
                tc::mbar_wait(full0 + 8 * s, (kb / kStages) & 1);
                tc::fence_after();
                const uint32_t a = tc::smem_u32(smem + s * kStageBytes), b = a + kABytes;
#pragma unroll
                for (int k = 0; k < BK / 32; ++k)   // K = 32 bytes per MMA
                    mma_i8(tmem_d, tc::desc_kmajor(a + 32 * k, 128), tc::desc_kmajor(b + 32 * k, 128),
                           (kb | k) != 0);
                tc::commit(empty0 + 8 * s);
            }
            tc::commit(tfull);
        }
    } else {   // epilogue warps 2..5: TMEM lane quarter warp % 4
        const int q = warp & 3;
        tc::mbar_wait(tfull, 0);
        tc::fence_after();
        const int64_t row = (int64_t)m_blk * BM + q * 32 + lane;
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            JACC_TMEM_LD_32(tmem_d + ((uint32_t)(q * 32) << 16) + c * 32, r);
            tc::wait_ld();
            if (row < ta) {
                const int64_t col0 = (int64_t)n_blk * BN + c * 32;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (col0 + j < tb) C[row * tb + col0 + j] = (int32_t)r[j];
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) {
        tc::fence_after();
        tc::dealloc_cols(tmem_d, kTmemCols);
    }
}

}  // namespace

size_t corr_ws_bytes(int64_t ta, int64_t tb, int64_t words) {
    const int64_t kp = round_up(words * 32 > 0 ? words * 32 : 1, BK);
    return (size_t)(round_up(ta > 0 ? ta : 1, BM) + round_up(tb > 0 ? tb : 1, BN)) * kp + 2048;
}

cudaError_t corr_popc_u32(const uint32_t *A, int64_t ta, const uint32_t *B, int64_t tb, int64_t words, int32_t *C,
                          void *ws, cudaStream_t st, int *launches) {
    if (ta <= 0 || tb <= 0) return cudaSuccess;
    if (words == 0) return cudaMemsetAsync(C, 0, (size_t)(ta * tb) * 4, st);
    const int64_t kp = round_up(words * 32, BK), tap = round_up(ta, BM), tbp = round_up(tb, BN);
    uint8_t *xa = (uint8_t *)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    uint8_t *xb = xa + tap * kp;
    const int grid_u = sm_count() * 8;
    unpack_kernel<<<grid_u, 256, 0, st>>>(A, ta, words, xa, tap, kp);
    unpack_kernel<<<grid_u, 256, 0, st>>>(B, tb, words, xb, tbp, kp);
    *launches += 2;
    CUtensorMap ma, mb;
    if (!tc::make_map_2d(&ma, xa, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, tap, kp, kp, BM, BK, 128) ||
        !tc::make_map_2d(&mb, xb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, tbp, kp, kp, BN, BK, 128))
        return cudaErrorInvalidValue;
    cudaError_t e = set_max_dyn_smem((const void *)corr_i8_kernel, kSmemBytes);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)(tbp / BN), (unsigned)(tap / BM));
    corr_i8_kernel<<<grid, kThreads, kSmemBytes, st>>>(ma, mb, C, ta, tb, (int)(kp / BK));
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
