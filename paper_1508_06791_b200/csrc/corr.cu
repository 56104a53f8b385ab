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
//      (when A and B are the same bitsets -- the paper's term-by-term matrix --
//      they are unpacked once);
//   2. GEMM: tcgen05.mma.cta_group::1.kind::i8 (u8 x u8 -> s32, exact),
//      128 x 256 output tile per CTA (48 KB of operands per 128-byte K block
//      for 4M multiply-adds: a 128 x 64 tile needed twice the bytes per MAC
//      and was bound by the SM's operand feed), K blocks staged by TMA (128B
//      swizzle) through a 4-stage mbarrier ring, accumulator in TMEM (256
//      columns), epilogue tcgen05.ld -> int32 stores;
//   3. split-K when the output has fewer tiles than SMs (1024 x 1024 = 32
//      tiles -> 4 splits): the splits of a tile run as one (1, 1, S) thread-
//      block cluster, each leaves its partial tile in its own shared memory,
//      and each CTA adds 1/S of the rows of all S partials over DSMEM, in
//      split order (integers: exact, independent of the split), straight
//      into C (45.7 -> 44.2 us at 1024 x 16384 with two unpacks: one launch
//      and 16 MB of partials fewer).  If no such cluster can be resident the
//      partials go to global memory and a small kernel adds them.
// The GEMM is launched with programmatic stream serialization: its CTAs do
// their prologue (barriers, TMEM allocation, tensor-map prefetch) while the
// unpack drains, and the TMA producer waits (griddepcontrol.wait) for the
// unpack grid before its first load (41.5 -> 36.9 us, two unpacks).
// One warp issues TMA, one thread issues the MMAs, four warps drain TMEM.
#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace jacc_k {
namespace {

constexpr int BM = 128, BN = 256, BK = 128;    // BK bytes = one 128 B swizzle row of u8
constexpr int kStages = 4;
constexpr int kABytes = BM * BK, kBBytes = BN * BK;
constexpr int kStageBytes = kABytes + kBBytes;  // 48 KB
constexpr int kThreads = 192;
constexpr int kTmemCols = BN;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
// kind::i8: D = s32 (c_format 2), A/B unsigned 8-bit (format 0), K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__host__ __device__ inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// bitsets [t x words] -> u8 [tp x kp]: byte d of row i = bit d%32 of word d/32.
// A warp expands 16 words into one contiguous 512-byte run per store: lane l
// writes bytes [16 l, 16 l + 16), the expansion of half (l & 1) of word l / 2
// -- every store instruction is fully coalesced.
__device__ __forceinline__ uint32_t expand4(uint32_t nib) {   // 4 bits -> 4 bytes (little endian)
    // nib x (1 + 2^7 + 2^14 + 2^21) places copies of the nibble at bits 0, 7,
    // 14, 21 (no carries: the copies do not overlap); bit k of copy k lands
    // on bit 8 k
    return ((nib & 0xFu) * 0x00204081u) & 0x01010101u;
}

template <typename I>   // index type: 32-bit when every index fits (the usual case), else 64-bit
__global__ void __launch_bounds__(256) unpack_kernel(const uint32_t *__restrict__ bits, I t, I words,
                                                     uint8_t *__restrict__ x, I tp, I kp) {
    constexpr int U = 4;   // runs per warp per pass: their loads are issued together
    // the GEMM (launched with programmatic stream serialization) may start its
    // prologue now; it waits (griddepcontrol.wait) for this grid's completion
    // and memory flush before its first TMA load of the unpacked rows
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x & 31;
    const I rpr = (kp + 511) / 512;    // kp is a multiple of 128: a row's last run may be partial
    const I total = tp * rpr;
    const I warp0 = (I)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const I nwarps = (I)(((int64_t)gridDim.x * blockDim.x) >> 5);
    for (I q0 = warp0; q0 < total; q0 += U * nwarps) {
        uint32_t v[U];
        I dst[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const I q = q0 + u * nwarps;
            const I r = q / rpr, byte = (q - r * rpr) * 512 + 16 * lane, w = byte / 32;
            ok[u] = q < total && byte < kp;
            dst[u] = r * kp + byte;
            v[u] = (ok[u] && r < t && w < words) ? __ldg(bits + (int64_t)r * words + w) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            const uint32_t h = (lane & 1) ? v[u] >> 16 : v[u];
            *(uint4 *)(x + (int64_t)dst[u]) = make_uint4(expand4(h), expand4(h >> 4), expand4(h >> 8), expand4(h >> 12));
        }
    }
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accum));
}

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {   // all threads of every CTA in the cluster
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_relaxed() {   // ordering only: nothing is published
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ int4 ld_dsmem_v4(uint32_t local_addr, uint32_t rank) {
    uint32_t a;
    int4 v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(local_addr), "r"(rank));
    asm volatile("ld.shared::cluster.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
    return v;
}

// Split-K partial tiles summed on chip: with a (1, 1, splits) cluster the
// splits of one output tile run as one cluster; each CTA leaves its 128 x 256
// int32 partial in its own (drained) ring memory, and after a cluster barrier
// CTA rank r adds rows [r BM / S, (r + 1) BM / S) of all S partials over DSMEM,
// in split order, and stores them to C.  Row stride 260 words: the epilogue's
// 16-byte stores of 32 rows hit 8 distinct 16-byte bank groups per wavefront.
constexpr int kTileStride = BN + 4;
constexpr int kMaxSplits = 8;   // a portable cluster
static_assert(BM * kTileStride * 4 <= kStages * kStageBytes, "partial tile fits in the ring");

// Rows [r0, r1) of the cluster's S partial tiles, summed in split order into
// C.  DSMEM loads are latency-bound (~1 us under this load): every thread
// issues the S loads of kU items before adding any (24 KB in flight per SM
// with 2 items took 4.6 us for a 1024^2 output; a load-add chain per split
// was slower still).
template <int S>
__device__ __forceinline__ void cluster_sum(uint32_t tile, int r0, int r1, int m_blk, int n_blk, int32_t *C,
                                            int64_t ta, int64_t tb, bool vec) {
    constexpr int kU = S <= 4 ? 4 : 2;
    const int nitems = (r1 - r0) * (BN / 4);
    for (int it0 = threadIdx.x; it0 < nitems; it0 += kU * kThreads) {
        int4 v[kU][S];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int it = it0 + u * kThreads;
            const uint32_t off = (uint32_t)((r0 + it / (BN / 4)) * kTileStride + (it % (BN / 4)) * 4) * 4;
#pragma unroll
            for (int sp = 0; sp < S; ++sp)
                if (it < nitems) v[u][sp] = ld_dsmem_v4(tile + off, (uint32_t)sp);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int it = it0 + u * kThreads;
            if (it >= nitems) continue;
            int4 acc = v[u][0];
#pragma unroll
            for (int sp = 1; sp < S; ++sp) {
                acc.x += v[u][sp].x; acc.y += v[u][sp].y; acc.z += v[u][sp].z; acc.w += v[u][sp].w;
            }
            const int lr = r0 + it / (BN / 4), lc = (it % (BN / 4)) * 4;
            const int64_t row = (int64_t)m_blk * BM + lr, col = (int64_t)n_blk * BN + lc;
            if (row >= ta || col >= tb) continue;
            int32_t *c = C + row * tb + col;
            if (vec) {
                *(int4 *)c = acc;
            } else {
                const int32_t a4[4] = {acc.x, acc.y, acc.z, acc.w};
                for (int k = 0; k < 4 && col + k < tb; ++k) c[k] = a4[k];
            }
        }
    }
}

// The same with 16-bit partials (each split's count is <= its K bits, so
// u16 holds it when a split spans <= 511 K blocks of 128): the partial rows
// are 256 u16 = 128 words, padded to kTileStride16; an item is 8 columns
// (one 16-byte DSMEM load per split) -- half the remote bytes of the 32-bit
// form, whose ~4.6 us of latency-bound DSMEM reads dominated the split-K
// epilogue at the paper's size.
constexpr int kTileStride16 = BN / 2 + 4;   // words per u16 partial row
template <int S>
__device__ __forceinline__ void cluster_sum16(uint32_t tile, int r0, int r1, int m_blk, int n_blk, int32_t *C,
                                              int64_t ta, int64_t tb, bool vec) {
    constexpr int kU = S <= 4 ? 4 : 2;
    const int nitems = (r1 - r0) * (BN / 8);
    for (int it0 = threadIdx.x; it0 < nitems; it0 += kU * kThreads) {
        int4 v[kU][S];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int it = it0 + u * kThreads;
            const uint32_t off = (uint32_t)((r0 + it / (BN / 8)) * kTileStride16 + (it % (BN / 8)) * 4) * 4;
#pragma unroll
            for (int sp = 0; sp < S; ++sp)
                if (it < nitems) v[u][sp] = ld_dsmem_v4(tile + off, (uint32_t)sp);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int it = it0 + u * kThreads;
            if (it >= nitems) continue;
            int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int sp = 0; sp < S; ++sp) {
                const uint32_t w[4] = {(uint32_t)v[u][sp].x, (uint32_t)v[u][sp].y, (uint32_t)v[u][sp].z,
                                       (uint32_t)v[u][sp].w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    acc[2 * h] += (int)(w[h] & 0xFFFFu);
                    acc[2 * h + 1] += (int)(w[h] >> 16);
                }
            }
            const int lr = r0 + it / (BN / 8), lc = (it % (BN / 8)) * 8;
            const int64_t row = (int64_t)m_blk * BM + lr, col = (int64_t)n_blk * BN + lc;
            if (row >= ta || col >= tb) continue;
            int32_t *c = C + row * tb + col;
            if (vec && col + 8 <= tb) {
                *(int4 *)c = make_int4(acc[0], acc[1], acc[2], acc[3]);
                *(int4 *)(c + 4) = make_int4(acc[4], acc[5], acc[6], acc[7]);
            } else {
                for (int k = 0; k < 8 && col + k < tb; ++k) c[k] = acc[k];
            }
        }
    }
}

// C tile (m_blk, n_blk) over K blocks [kb0, kb1).  ldc = tb and bounds
// checks when writing C directly; a padded [tap x tbp] partial (split
// blockIdx.z) when `part` is set; summed over the cluster's DSMEM when
// `csum` is set (cluster dims (1, 1, gridDim.z); 2: 16-bit partials).
__global__ void __launch_bounds__(kThreads, 1)
    corr_i8_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   int32_t *__restrict__ C, int64_t ta, int64_t tb, int num_kb, int32_t *__restrict__ part,
                   int64_t tap, int64_t tbp, int csum) {
    extern __shared__ uint8_t smem_raw[];
    // 1 KiB aligned by offset arithmetic on the shared array (through an integer
    // the compiler loses the address space: generic stores in the epilogue)
    uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *bars = (uint64_t *)(smem + kStages * kStageBytes);
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kStages + 1);
    const uint32_t full0 = tc::smem_u32(bars), empty0 = tc::smem_u32(bars + kStages),
                   tfull = tc::smem_u32(bars + 2 * kStages);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_blk = blockIdx.y, n_blk = blockIdx.x;
    const int per = (num_kb + gridDim.z - 1) / gridDim.z;
    const int kb0 = blockIdx.z * per, kb1 = min(num_kb, kb0 + per);
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
            asm volatile("griddepcontrol.wait;" ::: "memory");   // the unpack grid has completed
            for (int i = 0; i < kb1 - kb0; ++i) {
                const int s = i % kStages, kb = kb0 + i;
                tc::mbar_wait(empty0 + 8 * s, ((i / kStages) & 1) ^ 1);
                uint8_t *st = smem + s * kStageBytes;
                tc::mbar_expect_tx(full0 + 8 * s, kStageBytes);
                tc::tma_load_2d(tc::smem_u32(st), &map_a, kb * BK, m_blk * BM, full0 + 8 * s);
                tc::tma_load_2d(tc::smem_u32(st + kABytes), &map_b, kb * BK, n_blk * BN, full0 + 8 * s);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {   // MMA issuer
            for (int i = 0; i < kb1 - kb0; ++i) {
                const int s = i % kStages;
                tc::mbar_wait(full0 + 8 * s, (i / kStages) & 1);
                tc::fence_after();
                const uint32_t a = tc::smem_u32(smem + s * kStageBytes), b = a + kABytes;
#pragma unroll
                for (int k = 0; k < BK / 32; ++k)   // K = 32 bytes per MMA
                    mma_i8(tmem_d, tc::desc_kmajor(a + 32 * k, 128), tc::desc_kmajor(b + 32 * k, 128),
                           (i | k) != 0);
                tc::commit(empty0 + 8 * s);
            }
            tc::commit(tfull);
        }
    } else {   // epilogue warps 2..5: TMEM lane quarter warp % 4
        const int q = warp & 3;
        tc::mbar_wait(tfull, 0);
        tc::fence_after();
        const int64_t row = (int64_t)m_blk * BM + q * 32 + lane;
        int32_t *prow = part ? part + ((int64_t)blockIdx.z * tap + row) * tbp : nullptr;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            JACC_TMEM_LD_32(tmem_d + ((uint32_t)(q * 32) << 16) + c * 32, r);
            tc::wait_ld();
            const int64_t col0 = (int64_t)n_blk * BN + c * 32;
            if (csum == 2) {   // u16 partial tile (per-split counts < 2^16) into the drained ring
                uint32_t *trow = (uint32_t *)smem + (q * 32 + lane) * kTileStride16 + c * 16;
#pragma unroll
                for (int j = 0; j < 32; j += 8)
                    *(uint4 *)(trow + j / 2) = make_uint4(r[j] | (r[j + 1] << 16), r[j + 2] | (r[j + 3] << 16),
                                                          r[j + 4] | (r[j + 5] << 16), r[j + 6] | (r[j + 7] << 16));
            } else if (csum) {   // partial tile into this CTA's drained ring memory
                int32_t *trow = (int32_t *)smem + (q * 32 + lane) * kTileStride + c * 32;
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *(int4 *)(trow + j) = make_int4((int)r[j], (int)r[j + 1], (int)r[j + 2], (int)r[j + 3]);
            } else if (prow) {   // padded partial tile: 16-byte stores, no bounds
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *(int4 *)(prow + col0 + j) = make_int4((int)r[j], (int)r[j + 1], (int)r[j + 2], (int)r[j + 3]);
            } else if (row < ta) {
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
    if (csum) {
        cluster_sync();   // every split's partial tile is in its CTA's shared memory
        const int S = (int)gridDim.z, rank = (int)cluster_rank();
        const int r0 = rank * BM / S, r1 = (rank + 1) * BM / S;
        const uint32_t tile = tc::smem_u32(smem);
        const bool vec = (tb & 3) == 0 && (((uintptr_t)C) & 15) == 0;
        if (csum == 2) {
            switch (S) {
                case 2: cluster_sum16<2>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
                case 3: cluster_sum16<3>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
                case 4: cluster_sum16<4>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
                case 5: cluster_sum16<5>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
                case 6: cluster_sum16<6>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
                case 7: cluster_sum16<7>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
                default: cluster_sum16<8>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
            }
        } else switch (S) {   // the split count as a constant: every load of a pass in flight at once
            case 2: cluster_sum<2>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
            case 3: cluster_sum<3>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
            case 4: cluster_sum<4>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
            case 5: cluster_sum<5>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
            case 6: cluster_sum<6>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
            case 7: cluster_sum<7>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
            default: cluster_sum<8>(tile, r0, r1, m_blk, n_blk, C, ta, tb, vec); break;
        }
        cluster_sync_relaxed();   // no CTA leaves while a peer still reads its tile (loads done)
    }
}

// ---------------------------------------------------------------- CTA pair
// The same GEMM on 256 x 256 output tiles computed by a CTA PAIR
// (tcgen05.mma.cta_group::2.kind::i8, M = 256, N = 256, K = 32): CTA x of the
// pair stages A rows [128 x, 128 x + 128) and B rows (output columns)
// [128 x, 128 x + 128) of the tile, the leader's single thread issues the
// MMAs, which read both CTAs' shared memory and leave output rows
// [128 x, ...) in CTA x's TMEM.  Per SM and 128-byte K block the operands
// are 32 KB instead of 48 KB: the 1-SM kernel was bound by that ingest
// (655 cycles per K block, ~75 B/clk/SM).  Both CTAs' TMA loads complete on
// the LEADER's full barrier (cta_group::2 TMA, mbarrier in the peer CTA);
// the MMA commits arrive on both CTAs' empty barriers (multicast).
// Split-K: a (2, 1, S) cluster, rank = x + 2 z; CTA (x, z) adds rows
// [r0, r1) of the S partials with the same x over DSMEM, in split order.
constexpr int kHalfN = BN / 2;
constexpr int kStage2 = BM * BK + kHalfN * BK;   // 32 KB
constexpr int kStages2 = 6;
constexpr int kSmem2 = kStages2 * kStage2 + 1024 + 256;
static_assert(BM * kTileStride * 4 <= kStages2 * kStage2, "partial tile fits in the ring");
constexpr uint32_t kIdesc2 = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)((2 * BM) >> 4) << 24);

__device__ __forceinline__ void mma_i8_pair(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc2), "r"(accum));
}
// arrive on the barrier at `bar` in both CTAs of the pair (cluster ranks
// leader, leader + 1) once the MMAs issued so far have completed
__device__ __forceinline__ void commit_pair(uint32_t bar, uint32_t leader) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            bar),
        "h"((uint16_t)(3u << leader))
        : "memory");
}
// 2-D TMA whose completion is counted on the pair leader's mbarrier (cluster
// rank `leader`: with a (2, 1, S) cluster the pairs are ranks 2z, 2z + 1)
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap *map, int x, int y, uint32_t bar,
                                                 uint32_t leader) {
    uint32_t lb;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(lb) : "r"(bar), "r"(leader));
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(lb)
        : "memory");
}

template <int S>
__device__ __forceinline__ void cluster_sum_pair(uint32_t tile, int r0, int r1, int x, int m_blk2, int n_blk, int32_t *C,
                                                 int64_t ta, int64_t tb, bool vec) {
    constexpr int kU = S <= 4 ? 4 : 2;
    const int nitems = (r1 - r0) * (BN / 4);
    for (int it0 = threadIdx.x; it0 < nitems; it0 += kU * kThreads) {
        int4 v[kU][S];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int it = it0 + u * kThreads;
            const uint32_t off = (uint32_t)((r0 + it / (BN / 4)) * kTileStride + (it % (BN / 4)) * 4) * 4;
#pragma unroll
            for (int sp = 0; sp < S; ++sp)
                if (it < nitems) v[u][sp] = ld_dsmem_v4(tile + off, (uint32_t)(x + 2 * sp));
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const int it = it0 + u * kThreads;
            if (it >= nitems) continue;
            int4 acc = v[u][0];
#pragma unroll
            for (int sp = 1; sp < S; ++sp) {
                acc.x += v[u][sp].x; acc.y += v[u][sp].y; acc.z += v[u][sp].z; acc.w += v[u][sp].w;
            }
            const int lr = r0 + it / (BN / 4), lc = (it % (BN / 4)) * 4;
            const int64_t row = (int64_t)m_blk2 * 2 * BM + x * BM + lr, col = (int64_t)n_blk * BN + lc;
            if (row >= ta || col >= tb) continue;
            int32_t *c = C + row * tb + col;
            if (vec) {
                *(int4 *)c = acc;
            } else {
                const int32_t a4[4] = {acc.x, acc.y, acc.z, acc.w};
                for (int k = 0; k < 4 && col + k < tb; ++k) c[k] = a4[k];
            }
        }
    }
}

// grid (2 * tbp / BN, tap / (2 BM), S); cluster (2, 1, S)
__global__ void __launch_bounds__(kThreads, 1)
    corr_i8_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                        int32_t *__restrict__ C, int64_t ta, int64_t tb, int num_kb) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t *bars = (uint64_t *)(smem + kStages2 * kStage2);
    uint32_t *tmem_slot = (uint32_t *)(bars + 2 * kStages2 + 1);
    const uint32_t full0 = tc::smem_u32(bars), empty0 = tc::smem_u32(bars + kStages2),
                   tfull = tc::smem_u32(bars + 2 * kStages2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int x = (int)(blockIdx.x & 1);           // rank in the pair (cluster x)
    const uint32_t leader = cluster_rank() & ~1u;  // the pair's even cluster rank (= 2 z)
    const int n_blk = blockIdx.x >> 1, m_blk2 = blockIdx.y;
    const int S = (int)gridDim.z;
    const int per = (num_kb + S - 1) / S;
    const int kb0 = blockIdx.z * per, kb1 = min(num_kb, kb0 + per);
    if (warp == 0 && lane == 0) {
        tc::tma_prefetch(&map_a);
        tc::tma_prefetch(&map_b);
        for (int s = 0; s < kStages2; ++s) {
            tc::mbar_init(full0 + 8 * s, 1);
            tc::mbar_init(empty0 + 8 * s, 1);
        }
        tc::mbar_init(tfull, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc::fence_before();
    cluster_sync();    // barriers of every CTA initialised before any remote arrive / complete_tx
    tc::fence_after();
    const uint32_t tmem_d = *tmem_slot;
    if (warp == 0) {
        if (lane == 0) {   // TMA producer (each CTA): its A rows and its B rows, counted on the leader's barrier
            asm volatile("griddepcontrol.wait;" ::: "memory");   // the unpack grid has completed
            for (int i = 0; i < kb1 - kb0; ++i) {
                const int s = i % kStages2, kb = kb0 + i;
                tc::mbar_wait(empty0 + 8 * s, ((i / kStages2) & 1) ^ 1);
                uint8_t *st = smem + s * kStage2;
                if (x == 0) tc::mbar_expect_tx(full0 + 8 * s, 2 * kStage2);
                tma_load_2d_pair(tc::smem_u32(st), &map_a, kb * BK, m_blk2 * 2 * BM + x * BM, full0 + 8 * s,
                                 leader);
                tma_load_2d_pair(tc::smem_u32(st + BM * BK), &map_b, kb * BK, n_blk * BN + x * kHalfN,
                                 full0 + 8 * s, leader);
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && x == 0) {   // MMA issuer: the leader's single thread
            for (int i = 0; i < kb1 - kb0; ++i) {
                const int s = i % kStages2;
                tc::mbar_wait(full0 + 8 * s, (i / kStages2) & 1);
                tc::fence_after();
                const uint32_t a = tc::smem_u32(smem + s * kStage2), b = a + BM * BK;
#pragma unroll
                for (int k = 0; k < BK / 32; ++k)
                    mma_i8_pair(tmem_d, tc::desc_kmajor(a + 32 * k, 128), tc::desc_kmajor(b + 32 * k, 128),
                                (i | k) != 0);
                commit_pair(empty0 + 8 * s, leader);
            }
            commit_pair(tfull, leader);
        }
    } else {   // epilogue warps 2..5: TMEM lane quarter -> this CTA's partial tile in its drained ring
        const int q = warp & 3;
        tc::mbar_wait(tfull, 0);
        tc::fence_after();
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            JACC_TMEM_LD_32(tmem_d + ((uint32_t)(q * 32) << 16) + c * 32, r);
            tc::wait_ld();
            int32_t *trow = (int32_t *)smem + (q * 32 + lane) * kTileStride + c * 32;
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *(int4 *)(trow + j) = make_int4((int)r[j], (int)r[j + 1], (int)r[j + 2], (int)r[j + 3]);
        }
    }
    tc::fence_before();
    cluster_sync();    // every CTA's partial tile is in its shared memory; all MMAs have completed
    if (warp == 1) {
        tc::fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(kTmemCols));
    }
    const int z = (int)blockIdx.z;
    const int r0 = z * BM / S, r1 = (z + 1) * BM / S;
    const uint32_t tile = tc::smem_u32(smem);
    const bool vec = (tb & 3) == 0 && (((uintptr_t)C) & 15) == 0;
    switch (S) {
        case 1: cluster_sum_pair<1>(tile, r0, r1, x, m_blk2, n_blk, C, ta, tb, vec); break;
        case 2: cluster_sum_pair<2>(tile, r0, r1, x, m_blk2, n_blk, C, ta, tb, vec); break;
        case 3: cluster_sum_pair<3>(tile, r0, r1, x, m_blk2, n_blk, C, ta, tb, vec); break;
        default: cluster_sum_pair<4>(tile, r0, r1, x, m_blk2, n_blk, C, ta, tb, vec); break;
    }
    cluster_sync_relaxed();   // no CTA leaves while a peer still reads its tile
}

// C[i][j] = sum over splits of the partial tiles, in split order (exact).
// One row per blockIdx.y; 16-byte loads of the padded partials.
__global__ void __launch_bounds__(256) split_sum_kernel(const int32_t *__restrict__ part, int splits, int64_t tap,
                                                        int64_t tbp, int32_t *__restrict__ C, int64_t ta,
                                                        int64_t tb) {
    const int64_t i = blockIdx.y;
    const int64_t j0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (j0 >= tb) return;
    int4 acc = make_int4(0, 0, 0, 0);
    for (int s = 0; s < splits; ++s) {
        const int4 v = __ldg((const int4 *)(part + ((int64_t)s * tap + i) * tbp + j0));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    int32_t *c = C + i * tb + j0;
    if (j0 + 4 <= tb && (((uintptr_t)c) & 15) == 0) {
        *(int4 *)c = acc;
    } else {
        const int32_t a[4] = {acc.x, acc.y, acc.z, acc.w};
        for (int k = 0; k < 4 && j0 + k < tb; ++k) c[k] = a[k];
    }
}

// K splits: enough CTAs to cover the SMs, each split >= 8 K blocks.
int corr_splits(int64_t ta, int64_t tb, int64_t words) {
    const int64_t tiles = (round_up(ta, BM) / BM) * (round_up(tb, BN) / BN);
    const int64_t num_kb = round_up(words * 32 > 0 ? words * 32 : 1, BK) / BK;
    int64_t s = sm_count() / (tiles > 0 ? tiles : 1);
    if (s > num_kb / 8) s = num_kb / 8;
    return (int)(s < 1 ? 1 : s > kMaxSplits ? kMaxSplits : s);   // a portable cluster
}

}  // namespace

size_t corr_ws_bytes(int64_t ta, int64_t tb, int64_t words) {
    const int64_t kp = round_up(words * 32 > 0 ? words * 32 : 1, BK);
    const int64_t tap = round_up(ta > 0 ? ta : 1, BM), tbp = round_up(tb > 0 ? tb : 1, BN);
    const int splits = corr_splits(ta, tb, words);
    return (size_t)(tap + tbp) * kp + 2048 + (splits > 1 ? (size_t)splits * tap * tbp * 4 + 1024 : 0);
}

cudaError_t corr_popc_u32(const uint32_t *A, int64_t ta, const uint32_t *B, int64_t tb, int64_t words, int32_t *C,
                          void *ws, cudaStream_t st, int *launches) {
    if (ta <= 0 || tb <= 0) return cudaSuccess;
    if (words == 0) return cudaMemsetAsync(C, 0, (size_t)(ta * tb) * 4, st);
    const int64_t kp = round_up(words * 32, BK), tap = round_up(ta, BM), tbp = round_up(tb, BN);
    uint8_t *xa = (uint8_t *)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    uint8_t *xb = xa + tap * kp;
    const int grid_u = sm_count() * 8;
    const bool same = A == B && ta == tb;   // C = X X^T: one unpacked copy serves both operands
    const bool i32 = (tap > tbp ? tap : tbp) * kp < (1ll << 31);
    auto unpack = [&](const uint32_t *bits, int64_t t, uint8_t *x, int64_t tp) {
        if (i32)
            unpack_kernel<int32_t><<<grid_u, 256, 0, st>>>(bits, (int32_t)t, (int32_t)words, x, (int32_t)tp, (int32_t)kp);
        else
            unpack_kernel<int64_t><<<grid_u, 256, 0, st>>>(bits, t, words, x, tp, kp);
        ++*launches;
    };
    unpack(A, ta, xa, same ? tbp : tap);
    if (same)
        xb = xa;
    else
        unpack(B, tb, xb, tbp);
    CUtensorMap ma, mb;
    if (!tc::make_map_2d(&ma, xa, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, tap, kp, kp, BM, BK, 128) ||
        !tc::make_map_2d(&mb, xb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, tbp, kp, kp, BN, BK, 128))
        return cudaErrorInvalidValue;
    cudaError_t e;
    {   // CTA pairs on 256 x 256 tiles, split-K in a (2, 1, S <= 4) cluster; A rows
        // past the unpacked tap come from TMA's zero fill
        const int64_t tap2 = round_up(ta, 2 * BM), num_kb = kp / BK;
        const int64_t pairs = (tap2 / (2 * BM)) * (tbp / BN);
        int64_t S = sm_count() / (2 * pairs);
        if (S > num_kb / 8) S = num_kb / 8;
        S = S < 1 ? 1 : S > 4 ? 4 : S;
        // Only when the pairs fill at least half the SMs with <= 2 splits:
        // with fewer tiles the split-K clusters of 8 CTAs (2 x 4) are not all
        // co-resident (measured 1024 x 131072: 188 us vs 128 for the 1-SM
        // kernel's (1, 1, 4) clusters); those shapes keep the 1-SM kernel.
        const bool use_pair = 2 * pairs * (S < 2 ? S : 2) >= sm_count() / 2;
        if (S > 2) S = 2;
        CUtensorMap pa, pb;
        if (use_pair &&
            tc::make_map_2d(&pa, xa, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, same ? tbp : tap, kp, kp, BM, BK, 128) &&
            tc::make_map_2d(&pb, xb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, tbp, kp, kp, kHalfN, BK, 128) &&
            tap2 / (2 * BM) <= 65535) {
            e = set_max_dyn_smem((const void *)corr_i8_pair_kernel, kSmem2);
            if (e != cudaSuccess) return e;
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = (unsigned)S;
            attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[1].val.programmaticStreamSerializationAllowed = 1;
            cfg.gridDim = dim3((unsigned)(2 * (tbp / BN)), (unsigned)(tap2 / (2 * BM)), (unsigned)S);
            cfg.blockDim = dim3(kThreads);
            cfg.dynamicSmemBytes = kSmem2;
            cfg.stream = st;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (max_active_clusters((const void *)corr_i8_pair_kernel, &cfg) >= (S > 1 ? pairs : 1)) {
                cfg.numAttrs = 2;
                e = cudaLaunchKernelEx(&cfg, corr_i8_pair_kernel, (CUtensorMap)pa, (CUtensorMap)pb, C, ta, tb,
                                       (int)num_kb);
                ++*launches;
                if (e != cudaSuccess) return e;
                return cudaGetLastError();
            }
        }
    }
    e = set_max_dyn_smem((const void *)corr_i8_kernel, kSmemBytes);
    if (e != cudaSuccess) return e;
    const int splits = corr_splits(ta, tb, words);
    dim3 grid((unsigned)(tbp / BN), (unsigned)(tap / BM), (unsigned)splits);
    if (splits > 1) {   // split tiles summed over DSMEM when a (1, 1, splits) cluster fits
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = (unsigned)splits;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // overlap the prologue with the unpack
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmemBytes;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;   // the occupancy query takes the cluster shape only
        if (max_active_clusters((const void *)corr_i8_kernel, &cfg) > 0) {   // cached per shape
            cfg.numAttrs = 2;
            // 16-bit partials when every split's count fits (<= 511 K blocks of 128 bits per split)
            const int per = (int)((kp / BK + splits - 1) / splits);
            e = cudaLaunchKernelEx(&cfg, corr_i8_kernel, (CUtensorMap)ma, (CUtensorMap)mb, C, ta, tb, (int)(kp / BK),
                                   (int32_t *)nullptr, tap, tbp, per * BK <= 65535 ? 2 : 1);
            ++*launches;
            if (e != cudaSuccess) return e;
            return cudaGetLastError();
        }
    }
    int32_t *part = nullptr;
    if (splits > 1)
        part = (int32_t *)(((uintptr_t)(xb + tbp * kp) + 1023) & ~(uintptr_t)1023);
    corr_i8_kernel<<<grid, kThreads, kSmemBytes, st>>>(ma, mb, C, ta, tb, (int)(kp / BK), part, tap, tbp, 0);
    ++*launches;
    if (part) {
        split_sum_kernel<<<dim3((unsigned)((tb + 1023) / 1024), (unsigned)ta), 256, 0, st>>>(part, splits, tap, tbp,
                                                                                            C, ta, tb);
        ++*launches;
    }
    return cudaGetLastError();
}

}  // namespace jacc_k
