// sgemm_tcgen05.cu -- Dense matrix multiply (§4.2, P:484-485, P:525:
// "SGEMM"), C = A.B, row-major fp32, beta = 0 (reading R13), on the sm_100a
// 5th-generation tensor cores with the 3xTF32 split (JACC_SGEMM_3XTF32):
//
//   x = x_hi + x_lo,  x_hi = x with the low 13 mantissa bits cleared (exactly
//   representable in TF32), x_lo = x - x_hi (exact in fp32);
//   A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi     (A_lo.B_lo ~ 2^-22 dropped)
//
// accumulated in fp32 in TMEM.  It is used because it meets the north_star
// tolerance (1e-4 vs the fp64 oracle; DESIGN.md §SGEMM shows 1xTF32 does not
// on signed inputs).
//
// Two paths, the same three MMAs in the same order (bitwise-equal results,
// tested):
//   * default (16-byte aligned A, B and row strides): gemm_3xtf32_pair_kernel
//     -- a CTA pair per 256 x 256 tile (tcgen05 cta_group::2), raw A and B
//     tiles by TMA (B row-major = MN-major operand, no transpose), the hi
//     operand is the raw tile (the tensor core reads only the TF32 bits),
//     x_lo computed in shared memory by the epilogue warps; no pre-pass;
//   * fallback: split_a / split_bt write padded K-major hi/lo copies, then
//     gemm_3xtf32_kernel -- one 128 x 256 tile per CTA:
//        warp 0     TMA producer: per 16-wide K block, 4 boxes (A_hi, A_lo:
//                   128x16; B_hi, B_lo: 256x16) into a 4-stage mbarrier ring
//                   (48 KB per stage), 64B-swizzled;
//        warp 1     TMEM allocator + single-thread MMA issuer: per K block
//                   2 k-steps x 3 tcgen05.mma.cta_group::1.kind::tf32
//                   (M=128, N=256, K=8), D in TMEM: two 256-column fp32
//                   accumulators used alternately per 256-wide K chunk;
//                   tcgen05.commit frees the smem stage / signals the epilogue;
//        warps 2..9 epilogue: every 256 K, tcgen05.ld 32x32b.x32 TMEM ->
//                   registers, fp32 round-to-nearest accumulation of the
//                   chunk sums (see the kernel comment), then global stores
//                   (edge-guarded).
// Measured at 8192^3 (one B200, events): pre-split path 3.87 ms (split
// 0.25 ms + GEMM; 6.4 GB DRAM per task), pair path 3.50 ms (2.55 GB).
// Every output element accumulates its K products in the same order for any
// M/N blocking, so a row block of C computed on one rank equals the same rows
// computed on one GPU bit for bit.
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace jacc_k {
namespace {

// Swizzle width of the K-major smem tiles: one swizzle row = kSw bytes = BK
// tf32.  64 B rows give 48 KB stages, so 4 stages fit (128 B rows: 96 KB,
// only 2 stages -- the TMA latency then shows up as MMA bubbles).
constexpr int kSw = 64;
constexpr int BM = 128, BN = 256, BK = kSw / 4;
constexpr int kStages = kSw == 64 ? 4 : 2;
constexpr int kABytes = BM * BK * 4;
constexpr int kBBytes = BN * BK * 4;
constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;   // 48 KB (kSw 64) / 96 KB (kSw 128)
constexpr int kThreads = 320;                   // TMA warp, MMA warp, 8 epilogue warps
constexpr int kTmemCols = 512;                  // two 128 x 256 fp32 accumulators
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// ------------------------------------------------------------ PTX wrappers (tcgen05.cuh)
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::mbar_wait;
using tc::smem_u32;
using tc::tma_load_2d;
using tc::tma_prefetch;
__device__ __forceinline__ void tc_fence_before() { tc::fence_before(); }
__device__ __forceinline__ void tc_fence_after() { tc::fence_after(); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) { return tc::desc_kmajor(addr, kSw); }
// Instruction descriptor, kind::tf32: D f32, A/B tf32, both K-major, M=128, N=256.
constexpr uint32_t kIdesc = (1u << 4)                // c_format = F32
                            | (2u << 7)              // a_format = TF32
                            | (2u << 10)             // b_format = TF32
                            | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) { tc::commit(bar); }
#define TMEM_LD_32(taddr, r) JACC_TMEM_LD_32(taddr, r)

// ------------------------------------------------------------ split kernels
__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

__global__ void __launch_bounds__(256) split_a_kernel(const float *__restrict__ A, int64_t M, int64_t K, int64_t lda,
                                                      float *__restrict__ hi, float *__restrict__ lo, int64_t Mp,
                                                      int64_t Kp) {
    // grid.x covers Kp in chunks of 1024 (4 per thread), rows stride over grid.y
    const int64_t k = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (k >= Kp) return;
    for (int64_t r = blockIdx.y; r < Mp; r += gridDim.y) {
        float x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = (r < M && k + j < K) ? A[r * lda + k + j] : 0.f;
        float4 h, l;
        h.x = tf32_hi(x[0]); h.y = tf32_hi(x[1]); h.z = tf32_hi(x[2]); h.w = tf32_hi(x[3]);
        l.x = x[0] - h.x; l.y = x[1] - h.y; l.z = x[2] - h.z; l.w = x[3] - h.w;
        *(float4 *)(hi + r * Kp + k) = h;
        *(float4 *)(lo + r * Kp + k) = l;
    }
}

// B (K x N, row stride ldb) -> hi/lo of B^T, [Np x Kp] row-major (K contiguous).
// 64 (k) x 64 (n) tile per 256-thread block through shared memory: each
// thread reads 4 x 16 B along n (rows of B) and writes 4 x 16 B along k (rows
// of B^T) for hi and for lo -- 128-bit accesses on both sides.
__global__ void __launch_bounds__(256) split_bt_kernel(const float *__restrict__ B, int64_t K, int64_t N, int64_t ldb,
                                                       float *__restrict__ hi, float *__restrict__ lo, int64_t Np,
                                                       int64_t Kp) {
    __shared__ float t[64][65];
    const int64_t k0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
    const bool vec_in = ((ldb & 3) == 0) && (((uintptr_t)B & 15) == 0) && n0 + 64 <= N && k0 + 64 <= K;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int q = threadIdx.x + 256 * i;        // 1024 float4 of the 64 x 64 tile
        const int r = q >> 4, c4 = (q & 15) * 4;    // k row, n column
        const int64_t k = k0 + r;
        if (vec_in) {
            const float4 v = *(const float4 *)(B + k * ldb + n0 + c4);
            t[r][c4] = v.x; t[r][c4 + 1] = v.y; t[r][c4 + 2] = v.z; t[r][c4 + 3] = v.w;
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t n = n0 + c4 + j;
                t[r][c4 + j] = (k < K && n < N) ? B[k * ldb + n] : 0.f;
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int q = threadIdx.x + 256 * i;
        const int r = q >> 4, c4 = (q & 15) * 4;    // n row of B^T, k column
        const int64_t n = n0 + r, k = k0 + c4;
        if (n >= Np || k >= Kp) continue;           // Kp is a multiple of 16: k..k+3 < Kp
        float4 h, l;
        const float x0 = t[c4][r], x1 = t[c4 + 1][r], x2 = t[c4 + 2][r], x3 = t[c4 + 3][r];
        h.x = tf32_hi(x0); h.y = tf32_hi(x1); h.z = tf32_hi(x2); h.w = tf32_hi(x3);
        l.x = x0 - h.x; l.y = x1 - h.y; l.z = x2 - h.z; l.w = x3 - h.w;
        *(float4 *)(hi + n * Kp + k) = h;
        *(float4 *)(lo + n * Kp + k) = l;
    }
}

// ------------------------------------------------------------ GEMM kernel
// K is processed in chunks of kChunkKB K-blocks (256 K).  The tensor core
// accumulates one chunk into one of two TMEM buffers (its fp32 accumulation
// truncates: measured -1.6e-4 relative bias at K = 8192 when a whole K range
// stayed in TMEM); the epilogue warps promote each chunk sum into fp32
// registers with round-to-nearest adds while the MMAs fill the other buffer
// (the FP8 "promotion" pattern, here for TF32).  Bias per chunk ~ 96
// truncated adds ~ 5e-6 relative.
constexpr int kChunkKB = 256 / BK;
constexpr int kEpiWarps = 8;                        // 2 per TMEM lane quarter, 128 columns each

// Split-K (blockIdx.y = split, gridDim.y > 1 only when the output has fewer
// tiles than SMs): a split covers whole 256-wide K chunks and writes its
// partial tile to part[split][Mp][Np]; a second kernel adds the splits in
// order.  Every element's sum is then ((chunks of split 0) + (chunks of
// split 1)) + ... -- fixed for a given shape, but not the unsplit order, so
// row blocks are bitwise-equal across shardings only when neither splits.
__global__ void __launch_bounds__(kThreads, 1)
    gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                       const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                       float *__restrict__ C, int64_t M, int64_t N, int64_t ldc, int num_kb, int num_m,
                       int num_n, float *__restrict__ part, int64_t Mp, int64_t Np) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *bars = (uint64_t *)(smem + kStages * kStageBytes);
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kStages + 4);
    const uint32_t full_bar0 = smem_u32(bars), empty_bar0 = smem_u32(bars + kStages),
                   tfull0 = smem_u32(bars + 2 * kStages), tempty0 = smem_u32(bars + 2 * kStages + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // Grouped raster: consecutive CTAs walk kGroupM M-tiles for each N-tile,
    // so a wave of 148 CTAs touches ~16 M-strips x ~9 N-strips of A/B instead
    // of ~5 M-strips x all 32 N-strips (B re-read from HBM every wave).
    constexpr int kGroupM = 16;
    const int pid = blockIdx.x;
    const int per_group = kGroupM * num_n;
    const int first_m = (pid / per_group) * kGroupM;
    const int gm = min(num_m - first_m, kGroupM);
    const int m_blk = first_m + (pid % per_group) % gm;
    const int n_blk = (pid % per_group) / gm;
    const int all_chunks = (num_kb + kChunkKB - 1) / kChunkKB;
    const int per_split = (all_chunks + gridDim.y - 1) / gridDim.y;
    const int c_begin = blockIdx.y * per_split, c_end = min(all_chunks, c_begin + per_split);
    const int kb_begin = c_begin * kChunkKB, kb_end = min(num_kb, c_end * kChunkKB);
    const int nchunks = c_end > c_begin ? c_end - c_begin : 0;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&map_ahi); tma_prefetch(&map_alo); tma_prefetch(&map_bhi); tma_prefetch(&map_blo);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full_bar0 + 8 * s, 1);
            mbar_init(empty_bar0 + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, kEpiWarps);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) {
        tc::alloc_cols(smem_u32(tmem_slot), kTmemCols);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {   // ---- TMA producer
            for (int kb = kb_begin; kb < kb_end; ++kb) {
                const int i = kb - kb_begin;
                const int s = i % kStages;
                const uint32_t ph = (i / kStages) & 1;
                mbar_wait(empty_bar0 + 8 * s, ph ^ 1);
                uint8_t *st = smem + s * kStageBytes;
                const uint32_t fb = full_bar0 + 8 * s;
                mbar_expect_tx(fb, kStageBytes);
                tma_load_2d(smem_u32(st), &map_ahi, kb * BK, m_blk * BM, fb);
                tma_load_2d(smem_u32(st + kABytes), &map_alo, kb * BK, m_blk * BM, fb);
                tma_load_2d(smem_u32(st + 2 * kABytes), &map_bhi, kb * BK, n_blk * BN, fb);
                tma_load_2d(smem_u32(st + 2 * kABytes + kBBytes), &map_blo, kb * BK, n_blk * BN, fb);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // ---- MMA issuer (one thread for the whole CTA)
            for (int kb = kb_begin; kb < kb_end; ++kb) {
                const int i = kb - kb_begin;   // split-local: chunk = i / kChunkKB (splits start on chunks)
                const int s = i % kStages;
                const uint32_t ph = (i / kStages) & 1;
                const int chunk = i / kChunkKB, buf = chunk & 1;
                const bool first = (i % kChunkKB) == 0;
                const bool last = (i % kChunkKB) == kChunkKB - 1 || kb == kb_end - 1;
                const uint32_t tmem_d = tmem_base + buf * BN;
                if (first) {   // the epilogue has drained this buffer's previous chunk
                    mbar_wait(tempty0 + 8 * buf, ((chunk >> 1) & 1) ^ 1);
                    tc_fence_after();
                }
                mbar_wait(full_bar0 + 8 * s, ph);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * kStageBytes);
                const uint32_t a_hi = base, a_lo = base + kABytes, b_hi = base + 2 * kABytes,
                               b_lo = base + 2 * kABytes + kBBytes;
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {   // K = 8 tf32 = 32 B per MMA
                    const uint32_t off = k * 32;
                    mma_tf32(tmem_d, smem_desc(a_hi + off), smem_desc(b_hi + off), !(first && k == 0));
                    mma_tf32(tmem_d, smem_desc(a_hi + off), smem_desc(b_lo + off), 1);
                    mma_tf32(tmem_d, smem_desc(a_lo + off), smem_desc(b_hi + off), 1);
                }
                mma_commit(empty_bar0 + 8 * s);   // stage free once these MMAs have read it
                if (last) mma_commit(tfull0 + 8 * buf);   // chunk sum complete in TMEM
            }
        }
    } else {   // ---- epilogue warps 2..9: TMEM lane quarter q, column half h
        const int ew = warp - 2, q = warp & 3, h = ew >> 2;
        float acc[128];
#pragma unroll
        for (int i = 0; i < 128; ++i) acc[i] = 0.f;
        for (int chunk = 0; chunk < nchunks; ++chunk) {
            const int buf = chunk & 1;
            mbar_wait(tfull0 + 8 * buf, (chunk >> 1) & 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * BN + h * 128;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t r[32];
                TMEM_LD_32(taddr + j * 32, r);
                tc::wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[j * 32 + i] += __uint_as_float(r[i]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(tempty0 + 8 * buf);
        }
        const int64_t row = (int64_t)m_blk * BM + q * 32 + lane;
        if (part) {   // split partial: padded [Mp x Np], 16-byte stores, no bounds
            float *prow = part + ((int64_t)blockIdx.y * Mp + row) * Np + (int64_t)n_blk * BN + h * 128;
#pragma unroll
            for (int j = 0; j < 128; j += 4)
                *(float4 *)(prow + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        } else if (row < M) {
            float *crow = C + row * ldc;
            const int64_t col0 = (int64_t)n_blk * BN + h * 128;
            if (col0 + 128 <= N && ((ldc & 3) == 0) && (((uintptr_t)C & 15) == 0)) {
#pragma unroll
                for (int j = 0; j < 128; j += 4)
                    *(float4 *)(crow + col0 + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 128; ++j)
                    if (col0 + j < N) crow[col0 + j] = acc[j];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tc::dealloc_cols(tmem_base, kTmemCols);
    }
}

// ------------------------------------------------------------ in-kernel split, CTA pair (v2)
// The same 3xTF32 product without the split pre-pass, on 256 x 256 output
// tiles computed by a CTA PAIR (a (2,1,1) cluster, tcgen05 cta_group::2).
//
// * The raw fp32 tiles of A (K-major, as stored) and B (row-major K x N =
//   MN-major for the B operand: no transpose) arrive by TMA.  The tensor
//   core's kind::tf32 operand read takes only the TF32 bits of an fp32 word
//   (hw(x) = x & 0xFFFFE000 = x_hi -- pinned bitwise against the pre-split
//   path by tests/test_gpu_parity.py), so the raw tile IS the hi operand.
// * The epilogue warps, idle between chunk drains, write x_lo = x - x_hi of
//   every staged element next to it (same swizzled position: the split is
//   elementwise), then signal the leader CTA:
//       A.B ~= A.B(hw) + A.B_lo + A_lo.B
// * Pair: CTA r holds A rows [128 r, 128 r + 128) and B columns
//   [128 r, 128 r + 128) of the tile; the leader's single thread issues
//   tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 8), which reads both
//   CTAs' shared memory and writes rows [128 r, ...) of D into CTA r's TMEM.
//   Per SM and K block the tensor core reads 8 KB per MMA instead of 12 KB
//   (1-SM 128 x 256), which leaves shared-memory bandwidth for the split:
//   measured with 1-SM tiles, TMA writes + split + MMA reads (~187 B/clk)
//   oversubscribed the ~128 B/clk of shared memory (4.07 ms at 8192^3 vs
//   3.28 ms without the split); the pair needs ~125 B/clk.
// DRAM traffic: A and B once per tile (plus L2 misses), no hi/lo copies.
// Stage (K = 16) per CTA: A 8 KB + A_lo 8 KB (SW64 K-major) + B 8 KB + B_lo
// 8 KB (four 16 x 32 boxes, 128B swizzle with 32B atoms, MN-major).
constexpr int kPairBM = 2 * BM;                      // 256 rows per pair
constexpr int kHalfBN = BN / 2;                      // 128 B columns per CTA
constexpr int kBBox = 32;                            // B columns per TMA box (128 B rows)
constexpr int kBBoxBytes = BK * kBBox * 4;           // 2 KB
constexpr int kHBBytes = kHalfBN * BK * 4;           // 8 KB
constexpr int kStage2 = 2 * kABytes + 2 * kHBBytes;  // 32 KB
constexpr int kStages2 = 6;
constexpr int kSmem2 = kStages2 * kStage2 + 1024 + 256;
// kind::tf32, D f32, A K-major, B MN-major, M = 256, N = 256
constexpr uint32_t kIdesc2 = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(kPairBM >> 4) << 24);

// MN-major tf32 operands exist only in the 128-byte swizzle with 32-byte
// atoms (UMMA layout type SWIZZLE_128B_BASE32B = 1; TMA
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B): 32 fp32 along N per 128-byte row, the
// pattern repeating every 4 K rows (512 B).  (The plain 128B swizzle is
// accepted by the instruction and silently yields zeros -- measured.)
__device__ __forceinline__ uint64_t desc_b_mn(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFF) >> 4);              // start address
    d |= (uint64_t)(kBBoxBytes >> 4) << 16;              // LBO: next 32-column (MN) group = next box
    d |= (uint64_t)(512 >> 4) << 32;                     // SBO: next 4-row (K) swizzle atom
    d |= (uint64_t)1 << 46;                              // version 1
    d |= (uint64_t)1 << 61;                              // SWIZZLE_128B_BASE32B
    return d;
}

__device__ __forceinline__ void mma_tf32_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc2), "r"(accum));
}
// arrive on the mbarriers at this address in BOTH CTAs of the pair once the
// leader's MMAs issued so far have completed
__device__ __forceinline__ void commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            bar),
        "h"((uint16_t)3)
        : "memory");
}
// arrive on the leader CTA's (rank 0) mbarrier at the same offset.  The
// default (.release, .cta scope) form: an explicit .release.cluster arrive
// compiles to MEMBAR.ALL.GPU + ERRBAR per arrive, which measured 40 % of the
// split warps' stall samples and made the pair kernel 2x slower.
__device__ __forceinline__ void arrive_leader(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\t"
        "mapa.shared::cluster.u32 ra, %0, 0;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_3xtf32_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                            float *__restrict__ C, int64_t M, int64_t N, int64_t ldc, int num_kb, int num_m2,
                            int num_n, float *__restrict__ part, int64_t Mp, int64_t Np) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *bars = (uint64_t *)(smem + kStages2 * kStage2);
    uint32_t *tmem_slot = (uint32_t *)(bars + 3 * kStages2 + 4);
    // full: this CTA's TMA landed its raw tiles; empty: the pair's MMAs read
    // the stage (multicast commit); split: both CTAs wrote their lo tiles
    // (leader's, 16 arrivals); tfull / tempty: accumulator buffer handshake
    // (tempty: leader's, 16 arrivals)
    const uint32_t full_bar0 = smem_u32(bars), empty_bar0 = smem_u32(bars + kStages2),
                   split_bar0 = smem_u32(bars + 2 * kStages2), tfull0 = smem_u32(bars + 3 * kStages2),
                   tempty0 = smem_u32(bars + 3 * kStages2 + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cta_rank();
    constexpr int kGroupM = 8;                       // pair tiles (256 rows) per raster group
    const int pid = blockIdx.x >> 1;
    const int per_group = kGroupM * num_n;
    const int first_m = (pid / per_group) * kGroupM;
    const int gm = min(num_m2 - first_m, kGroupM);
    const int m_blk = first_m + (pid % per_group) % gm;
    const int n_blk = (pid % per_group) / gm;
    const int all_chunks = (num_kb + kChunkKB - 1) / kChunkKB;
    const int per_split = (all_chunks + gridDim.y - 1) / gridDim.y;
    const int c_begin = blockIdx.y * per_split, c_end = min(all_chunks, c_begin + per_split);
    const int kb_begin = c_begin * kChunkKB, kb_end = min(num_kb, c_end * kChunkKB);
    const int nchunks = c_end > c_begin ? c_end - c_begin : 0;
    const int nkb = kb_end > kb_begin ? kb_end - kb_begin : 0;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&map_a); tma_prefetch(&map_b);
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(full_bar0 + 8 * s, 1);
            mbar_init(empty_bar0 + 8 * s, 1);
            mbar_init(split_bar0 + 8 * s, 2 * kEpiWarps);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull0 + 8 * b, 1);
            mbar_init(tempty0 + 8 * b, 2 * kEpiWarps);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) {   // both CTAs' warp 1: one 2-SM allocation at the same TMEM address
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();    // barriers initialised in both CTAs before any remote arrive
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {   // ---- TMA producer (each CTA): its A rows and its B columns
            for (int i = 0; i < nkb; ++i) {
                const int kb = kb_begin + i, s = i % kStages2;
                mbar_wait(empty_bar0 + 8 * s, ((i / kStages2) & 1) ^ 1);
                uint8_t *st = smem + s * kStage2;
                const uint32_t fb = full_bar0 + 8 * s;
                mbar_expect_tx(fb, kABytes + kHBBytes);
                tma_load_2d(smem_u32(st), &map_a, kb * BK, m_blk * kPairBM + (int)rank * BM, fb);
                const uint32_t bdst = smem_u32(st + 2 * kABytes);
#pragma unroll
                for (int j = 0; j < kHalfBN / kBBox; ++j)
                    tma_load_2d(bdst + j * kBBoxBytes, &map_b, n_blk * BN + (int)rank * kHalfBN + j * kBBox,
                                kb * BK, fb);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {   // ---- MMA issuer: the leader's single thread
            for (int i = 0; i < nkb; ++i) {
                const int s = i % kStages2;
                const int chunk = i / kChunkKB, buf = chunk & 1;
                const bool first = (i % kChunkKB) == 0;
                const bool last = (i % kChunkKB) == kChunkKB - 1 || i == nkb - 1;
                const uint32_t tmem_d = tmem_base + buf * BN;
                if (first) {
                    mbar_wait(tempty0 + 8 * buf, ((chunk >> 1) & 1) ^ 1);
                    tc_fence_after();
                }
                mbar_wait(split_bar0 + 8 * s, (i / kStages2) & 1);
                tc_fence_after();
                const uint32_t base = smem_u32(smem + s * kStage2);
                const uint32_t a_raw = base, a_lo = base + kABytes, b_raw = base + 2 * kABytes,
                               b_lo = base + 2 * kABytes + kHBBytes;
#pragma unroll
                for (int k = 0; k < BK / 8; ++k) {
                    const uint32_t oa = k * 32, ob = k * 1024;   // A: 32 B along K; B: 8 rows of 128 B
                    mma_tf32_pair(tmem_d, smem_desc(a_raw + oa), desc_b_mn(b_raw + ob), !(first && k == 0));
                    mma_tf32_pair(tmem_d, smem_desc(a_raw + oa), desc_b_mn(b_lo + ob), 1);
                    mma_tf32_pair(tmem_d, smem_desc(a_lo + oa), desc_b_mn(b_raw + ob), 1);
                }
                commit_pair(empty_bar0 + 8 * s);
                if (last) commit_pair(tfull0 + 8 * buf);
            }
        }
    } else {   // ---- warps 2..9 (each CTA): split the staged tiles, drain the chunk sums
        const int ew = warp - 2, q = warp & 3, h = ew >> 2;
        float acc[128];
#pragma unroll
        for (int i = 0; i < 128; ++i) acc[i] = 0.f;
        int drained = 0;
        auto drain = [&](int chunk) {
            const int buf = chunk & 1;
            mbar_wait(tfull0 + 8 * buf, (chunk >> 1) & 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + buf * BN + h * 128;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t r[32];
                TMEM_LD_32(taddr + j * 32, r);
                tc::wait_ld();
#pragma unroll
                for (int t = 0; t < 32; ++t) acc[j * 32 + t] += __uint_as_float(r[t]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) arrive_leader(tempty0 + 8 * buf);
        };
        constexpr int kVec = (kABytes + kHBBytes) / 16;         // float4s to split per stage
        constexpr int kPer = kVec / (kEpiWarps * 32);           // 4 per thread
        const int et = ew * 32 + lane;
        for (int i = 0; i < nkb; ++i) {
            const int s = i % kStages2;
            mbar_wait(full_bar0 + 8 * s, (i / kStages2) & 1);
            uint8_t *st = smem + s * kStage2;
            float4 v[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int f = et + u * kEpiWarps * 32;           // float4 index over [A | B]
                const int off = f < kABytes / 16 ? f * 16 : 2 * kABytes + (f * 16 - kABytes);
                v[u] = *(const float4 *)(st + off);
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int f = et + u * kEpiWarps * 32;
                const int off = f < kABytes / 16 ? f * 16 + kABytes : 2 * kABytes + kHBBytes + (f * 16 - kABytes);
                float4 l;
                l.x = v[u].x - tf32_hi(v[u].x); l.y = v[u].y - tf32_hi(v[u].y);
                l.z = v[u].z - tf32_hi(v[u].z); l.w = v[u].w - tf32_hi(v[u].w);
                *(float4 *)(st + off) = l;
            }
            // generic-proxy stores -> visible to the tensor core (async proxy)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) arrive_leader(split_bar0 + 8 * s);
            // chunk c's MMAs need nothing more from this CTA once chunk c+1
            // is split: drain it now (the leader still has the staged stages
            // of chunk c+1 to issue)
            if ((i % kChunkKB) == kChunkKB - 1 && i / kChunkKB >= 1) drain(drained++);
        }
        while (drained < nchunks) drain(drained++);
        const int64_t row = (int64_t)m_blk * kPairBM + (int64_t)rank * BM + q * 32 + lane;
        if (part) {
            float *prow = part + ((int64_t)blockIdx.y * Mp + row) * Np + (int64_t)n_blk * BN + h * 128;
#pragma unroll
            for (int j = 0; j < 128; j += 4)
                *(float4 *)(prow + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
        } else if (row < M) {
            float *crow = C + row * ldc;
            const int64_t col0 = (int64_t)n_blk * BN + h * 128;
            if (col0 + 128 <= N && ((ldc & 3) == 0) && (((uintptr_t)C & 15) == 0)) {
#pragma unroll
                for (int j = 0; j < 128; j += 4)
                    *(float4 *)(crow + col0 + j) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 128; ++j)
                    if (col0 + j < N) crow[col0 + j] = acc[j];
            }
        }
    }
    tc_fence_before();
    cluster_sync_all();    // the leader's MMAs read both CTAs' smem: nobody leaves early
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
    }
}

// C = sum of the split partials, in split order.  One row per blockIdx.y,
// four columns per thread (16-byte partial loads; Np is a multiple of 256).
__global__ void __launch_bounds__(256) split_sum_f32_kernel(const float *__restrict__ part, int splits, int64_t Mp,
                                                            int64_t Np, float *__restrict__ C, int64_t M, int64_t N,
                                                            int64_t ldc) {
    const int64_t i = blockIdx.y;
    const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= M || j >= N) return;
    float4 acc = __ldg((const float4 *)(part + i * Np + j));
    for (int s = 1; s < splits; ++s) {
        const float4 v = __ldg((const float4 *)(part + ((int64_t)s * Mp + i) * Np + j));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    float *c = C + i * ldc + j;
    if (j + 4 <= N && (((uintptr_t)c) & 15) == 0) {
        *(float4 *)c = acc;
    } else {
        const float a[4] = {acc.x, acc.y, acc.z, acc.w};
        for (int k = 0; k < 4 && j + k < N; ++k) c[k] = a[k];
    }
}

// K splits for a grid of `tiles` output tiles: only when the tiles leave SMs
// idle; whole 256-wide chunks per split.
int sgemm_splits(int64_t tiles, int64_t Kp) {
    const int64_t chunks = (Kp / BK + kChunkKB - 1) / kChunkKB;
    const int sms = sm_count();
    if (tiles >= sms || chunks < 2) return 1;
    int64_t s = sms / tiles;
    if (s > chunks) s = chunks;
    if (s > 8) s = 8;
    // equal chunk counts per split (no empty trailing split)
    while (s > 1 && (chunks + s - 1) / s * (s - 1) >= chunks) --s;
    return (int)(s < 1 ? 1 : s);
}

// ------------------------------------------------------------ host side
bool make_map(CUtensorMap *m, const float *base, int64_t rows, int64_t kp, int box_rows) {
    return tc::make_map_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, rows, kp, kp * 4, box_rows, BK, kSw);
}

// JACC_SGEMM_V1=1: force the split pre-pass path (A/B comparisons only)
bool getenv_flag_v1() {
    static const bool v = [] { const char *e = getenv("JACC_SGEMM_V1"); return e && e[0] == '1'; }();
    return v;
}

}  // namespace

size_t sgemm_3xtf32_ws_bytes(const jacc_sgemm_params_t *p) {
    const int64_t Mp = round_up(p->M > 0 ? p->M : 1, BM), Np = round_up(p->N > 0 ? p->N : 1, BN),
                  Kp = round_up(p->K > 0 ? p->K : 1, BK);
    const int splits = sgemm_splits((Mp / BM) * (Np / BN), Kp);
    const size_t v1 = (size_t)(2 * Mp * Kp + 2 * Np * Kp) * 4 + 4096 + (splits > 1 ? (size_t)splits * Mp * Np * 4 + 1024 : 0);
    // the pair path needs only its split-K partials (alignment decides the
    // path at launch, so provide for both)
    const int64_t Mp2 = round_up(p->M > 0 ? p->M : 1, kPairBM);
    const int splits2 = sgemm_splits(2 * (Mp2 / kPairBM) * (Np / BN), Kp);
    const size_t v2 = splits2 > 1 ? (size_t)splits2 * Mp2 * Np * 4 + 1024 : 0;
    return v1 > v2 ? v1 : v2;
}

cudaError_t sgemm_3xtf32(const float *A, const float *B, float *C, const jacc_sgemm_params_t *p, void *ws,
                         cudaStream_t st, int *launches) {
    const int64_t M = p->M, N = p->N, K = p->K;
    if (M == 0 || N == 0) return cudaSuccess;
    if (K == 0)   // C = 0 (beta = 0): the M x N window only
        return cudaMemset2DAsync(C, (size_t)p->ldc * 4, 0, (size_t)N * 4, (size_t)M, st);
    const int64_t Mp = round_up(M, BM), Np = round_up(N, BN), Kp = round_up(K, BK);
    const int num_m = (int)(Mp / BM), num_n = (int)(Np / BN);
    const int splits = sgemm_splits((int64_t)num_m * num_n, Kp);
    // v2 (CTA pair, in-kernel split, no pre-pass): TMA straight from A and
    // B, which needs 16-byte aligned bases and row strides
    if (aligned16(A) && aligned16(B) && (p->lda & 3) == 0 && (p->ldb & 3) == 0 && !getenv_flag_v1()) {
        CUtensorMap m_a, m_b;
        if (tc::make_map_2d(&m_a, A, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, M, K, p->lda * 4, BM, BK, kSw) &&
            tc::make_map_2d_swz(&m_b, B, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, K, N, p->ldb * 4, BK, kBBox,
                                CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
            cudaError_t e = set_max_dyn_smem((const void *)gemm_3xtf32_pair_kernel, kSmem2);
            if (e != cudaSuccess) return e;
            const int64_t Mp2 = round_up(M, kPairBM);
            const int num_m2 = (int)(Mp2 / kPairBM);
            const int splits2 = sgemm_splits(2 * (int64_t)num_m2 * num_n, Kp);
            float *part = splits2 > 1 ? (float *)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023) : nullptr;
            gemm_3xtf32_pair_kernel<<<dim3(2 * num_m2 * num_n, splits2), kThreads, kSmem2, st>>>(
                m_a, m_b, C, M, N, p->ldc, (int)(Kp / BK), num_m2, num_n, part, Mp2, Np);
            ++*launches;
            if (part) {
                split_sum_f32_kernel<<<dim3((unsigned)((N + 1023) / 1024), (unsigned)M), 256, 0, st>>>(
                    part, splits2, Mp2, Np, C, M, N, p->ldc);
                ++*launches;
            }
            return cudaGetLastError();
        }
    }
    float *ahi = (float *)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    float *alo = ahi + Mp * Kp;
    float *bhi = alo + Mp * Kp;
    float *blo = bhi + Np * Kp;
    {
        dim3 g1((unsigned)((Kp + 1023) / 1024), (unsigned)(Mp < 65535 ? Mp : 65535));
        split_a_kernel<<<g1, 256, 0, st>>>(A, M, K, p->lda, ahi, alo, Mp, Kp);
        dim3 g2((unsigned)((Np + 63) / 64), (unsigned)((Kp + 63) / 64));
        split_bt_kernel<<<g2, 256, 0, st>>>(B, K, N, p->ldb, bhi, blo, Np, Kp);
        *launches += 2;
    }
    CUtensorMap m_ahi, m_alo, m_bhi, m_blo;
    if (!make_map(&m_ahi, ahi, Mp, Kp, BM) || !make_map(&m_alo, alo, Mp, Kp, BM) ||
        !make_map(&m_bhi, bhi, Np, Kp, BN) || !make_map(&m_blo, blo, Np, Kp, BN))
        return cudaErrorInvalidValue;
    cudaError_t e = set_max_dyn_smem((const void *)gemm_3xtf32_kernel, kSmemBytes);
    if (e != cudaSuccess) return e;
    float *part = splits > 1 ? (float *)(((uintptr_t)(blo + Np * Kp) + 1023) & ~(uintptr_t)1023) : nullptr;
    gemm_3xtf32_kernel<<<dim3(num_m * num_n, splits), kThreads, kSmemBytes, st>>>(
        m_ahi, m_alo, m_bhi, m_blo, C, M, N, p->ldc, (int)(Kp / BK), num_m, num_n, part, Mp, Np);
    ++*launches;
    if (part) {
        split_sum_f32_kernel<<<dim3((unsigned)((N + 1023) / 1024), (unsigned)M), 256, 0, st>>>(part, splits, Mp, Np,
                                                                                             C, M, N, p->ldc);
        ++*launches;
    }
    return cudaGetLastError();
}

}  // namespace jacc_k
