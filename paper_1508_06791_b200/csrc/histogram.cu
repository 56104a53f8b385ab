// histogram.cu -- Histogram (§4.2): "frequency counts for
// ... values, placing the results into 256 distinct bins"; the bins are an
// @Atomic(op=ADD) output (Table 1) updated "using shared memory
// atomic operations" and auto-zeroed.
//
// bins[k] += #{i : keys[i] == k} for 0 <= k < nbins; other keys are ignored
// (reading R11).  Integer counts: bit-exact by construction.
//
// sm_100a design (nbins <= 256), sized so the HBM read of 4 B/key binds:
//   * privatisation at the finest grain -- every LANE owns a private 16-bit
//     sub-histogram in shared memory, laid out word (bin/2)*32 + lane, half
//     bin%2.  A lane's word always sits in bank `lane`, so the 32 updates of
//     a warp never conflict, for ANY key distribution (uniform or all-equal);
//     the update is a shared-memory atomic add whose result is unused (no
//     dependency chain between a lane's keys).  Two warps share each
//     sub-histogram (lane l of both: still bank l), which halves the shared
//     memory per warp and lets 16 warps per SM stream keys instead of 12.
//   * keys stream in as 128-bit loads, 8 int4 per lane per chunk, with the
//     next chunk prefetched into registers while the current one is counted.
//   * before a 16-bit counter can overflow (every 1023 chunks of the pair:
//     <= 65472 keys per lane counter; both warps run the same trip count and
//     meet at a pair barrier) one warp of the pair folds the sub-histogram
//     into per-lane 32-bit register totals (lane l
//     owns bins 8l..8l+7; column reads are rotated so they stay
//     conflict-free) and clears them (an 8-bit form had to fold every 240
//     keys: 184 vs 182 us at 2^28);
//   * at the end the warps' totals are combined with shared-memory atomics
//     into one block histogram, added ONCE per block into a workspace
//     accumulator; the last block (grid ticket) writes the @Atomic bins --
//     assigned for a W output (the auto-zero, without a memset),
//     added for RW -- and re-zeroes the accumulator.
// nbins in (256, 4096]: a plain shared-memory-atomics block histogram.
//
// JACC_GRAPH_P2P fusion (reading R23): when the graph's next task is the
// allreduce of these bins, the same kernel finishes it -- the last block
// (the grid ticket in the peer window) writes the local bins, pushes them
// into every rank's window over NVLink, waits for the other ranks' rows and
// sums them in rank order (peer.cuh block_allreduce): one launch instead of
// histogram + NCCL.
#include "common.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace jacc_k {
namespace {

// 16-bit lane-private counters: word (bin/2)*32 + lane, half bin%2 -- 16 KB
// per sub-histogram, SHARED by the two warps of a pair (lane l of both warps
// owns bank l, so the sharing adds no bank conflict): 2 sub-histograms per
// 4-warp block, 4 blocks (16 warps) per SM.  One sub-histogram per warp
// capped the SM at 12 warps (16.5 KB each): 181 -> 168 us at 2^28 keys.
// A counter is folded before it can overflow -- every 1023 chunks of the
// pair (2 x 1023 x 32 = 65472 keys per lane counter) instead of every 240
// keys of the 8-bit form (whose fold cost ~0.5 shared op + ~1 ALU op per key).
constexpr int kWarps16 = 4;
constexpr int kBlock16 = kWarps16 * 32;
constexpr int kU16 = 8;                    // int4 per lane per chunk (32 keys)
constexpr int kChunk16 = 32 * kU16;
constexpr int kSubWords16 = 129 * 32;      // 256 bins / 2 per word + 1 dummy group, x 32 lanes
constexpr int kShare = 2;                  // warps per sub-histogram (lane l of each writes bank l)
constexpr int kFoldPair = 1023;            // 2 warps x 1023 chunks x 32 keys <= 65535 per lane counter
constexpr int kBlocksPerSm16 = 4;          // 34 KB of shared memory, 128 registers per thread
constexpr int kSmemBytes16 = (kWarps16 / kShare) * kSubWords16 * 4 + 256 * 4;

__device__ __forceinline__ void count_key16(unsigned *sub_lane_w, int k, unsigned nbins) {
    const unsigned kk = min((unsigned)k, nbins);
    atomicAdd(sub_lane_w + ((kk >> 1) << 5), 1u << ((kk & 1u) << 4));
}

// lane l folds bins 8l..8l+7 (word groups 4l..4l+3) over the 32 lanes' words
__device__ __forceinline__ void flush16(unsigned *sub, unsigned lane, unsigned tot[8]) {
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const unsigned g = 4 * lane + h;               // bins 2g, 2g+1
        unsigned lo = 0, hi = 0;
#pragma unroll 8
        for (unsigned c = 0; c < 32; ++c) {
            const unsigned v = sub[g * 32 + ((c + lane) & 31)];
            lo += v & 0xFFFFu;
            hi += v >> 16;
        }
        tot[2 * h] += lo;
        tot[2 * h + 1] += hi;
    }
    __syncwarp();
#pragma unroll 8
    for (int g = 0; g < 128; ++g) sub[g * 32 + lane] = 0u;
    __syncwarp();
}

// The blocks' histograms meet in a workspace accumulator (256 u32, kept
// zeroed between launches); the LAST block (grid ticket) stores bins =
// acc (W: the @Atomic output's auto-zero, without a memset node) or
// bins += acc (RW), re-zeroes acc and re-arms the ticket -- and, fused,
// completes the allreduce of the bins over the peer windows.
template <bool kPeer>
__global__ void __launch_bounds__(kBlock16) hist256_w16_kernel(const int4 *__restrict__ keys4, int64_t n4,
                                                               const int32_t *__restrict__ edge, int n_edge,
                                                               int32_t *__restrict__ bins, int nbins,
                                                               unsigned *__restrict__ acc, int assign, PeerOp pop) {
    extern __shared__ unsigned smem[];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned *sub = smem + (warp / kShare) * kSubWords16;
    unsigned *blockh = smem + (kWarps16 / kShare) * kSubWords16;
    if (warp % kShare == 0)
        for (int g = 0; g < 129; ++g) sub[g * 32 + lane] = 0u;
    for (int i = threadIdx.x; i < 256; i += kBlock16) blockh[i] = 0u;
    __syncthreads();
    unsigned tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int64_t nwarps = (int64_t)gridDim.x * kWarps16;
    const int64_t c0 = (int64_t)blockIdx.x * kWarps16 + warp;
    const int64_t nchunks = (n4 + kChunk16 - 1) / kChunk16;
    const int64_t trips = (nchunks + nwarps - 1) / nwarps;   // the same for every warp (pair barriers)
    int4 cur[kU16], nxt[kU16];
    auto load = [&](int64_t ch, int4 *dst) {
        if ((ch + 1) * kChunk16 <= n4) {
#pragma unroll
            for (int u = 0; u < kU16; ++u) dst[u] = ld_stream(keys4 + ch * kChunk16 + u * 32 + lane);
        } else {
#pragma unroll
            for (int u = 0; u < kU16; ++u) {
                const int64_t idx = ch * kChunk16 + u * 32 + lane;
                dst[u] = (ch < nchunks && idx < n4) ? ld_stream(keys4 + idx) : make_int4(-1, -1, -1, -1);
            }
        }
    };
    auto pair_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + warp / kShare), "n"(32 * kShare) : "memory"); };
    if (c0 < nchunks) load(c0, cur);
    for (int64_t k = 0; k < trips; ++k) {
        const int64_t c = c0 + k * nwarps;
        load(c + nwarps, nxt);
        if (c < nchunks) {
#pragma unroll
            for (int u = 0; u < kU16; ++u) {
                count_key16(sub + lane, cur[u].x, nbins);
                count_key16(sub + lane, cur[u].y, nbins);
                count_key16(sub + lane, cur[u].z, nbins);
                count_key16(sub + lane, cur[u].w, nbins);
            }
        }
        if ((k + 1) % kFoldPair == 0) {
            pair_sync();
            if (warp % kShare == 0) flush16(sub, lane, tot);
            pair_sync();
        }
#pragma unroll
        for (int u = 0; u < kU16; ++u) cur[u] = nxt[u];
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < n_edge; i += kBlock16) {
            const int k = edge[i];
            if ((unsigned)k < (unsigned)nbins) atomicAdd(&blockh[k], 1u);
        }
    }
    pair_sync();
    if (warp % kShare == 0) flush16(sub, lane, tot);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (tot[j]) atomicAdd(&blockh[8 * lane + j], tot[j]);
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += kBlock16)
        if (blockh[i]) atomicAdd(&acc[i], blockh[i]);
    unsigned *ticket = acc + 256;
    __shared__ bool last;
    if (kPeer) {
        last = peer::grid_last(pop.ctx, pop.slot);
    } else {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
    }
    if (!last) return;
    __threadfence();
    for (int i = threadIdx.x; i < nbins; i += kBlock16) {
        const int v = (int)__ldcg(acc + i);
        bins[i] = assign ? v : bins[i] + v;
        acc[i] = 0u;
    }
    if (!kPeer && threadIdx.x == 0) *ticket = 0u;   // re-arm (stream-ordered before the next launch)
    if (kPeer) peer::block_allreduce<int>(pop.ctx, pop.slot, (size_t)pop.off, bins, nbins);
}

// nbins in (256, 4096]: one shared 32-bit histogram per block, smem atomics.
__global__ void __launch_bounds__(256) hist_big_kernel(const int32_t *__restrict__ keys, int64_t n,
                                                       int32_t *__restrict__ bins, int nbins) {
    extern __shared__ unsigned h[];
    for (int i = threadIdx.x; i < nbins; i += blockDim.x) h[i] = 0u;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const int k = __ldg(keys + i);
        if ((unsigned)k < (unsigned)nbins) atomicAdd(&h[k], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nbins; i += blockDim.x)
        if (h[i]) atomicAdd(&bins[i], (int)h[i]);
}

}  // namespace

size_t histogram_ws_bytes(int64_t, int) { return 257 * sizeof(unsigned); }   // acc[256] + ticket

cudaError_t histogram_i32(const int32_t *keys, int64_t n, int32_t *bins, int nbins, void *ws, const jacc_schedule_t *s,
                          cudaStream_t st, int *launches, const PeerOp *pop, bool assign) {
    if (pop && (n <= 0 || nbins > 256)) return cudaErrorInvalidValue;   // the runtime only fuses these
    if (n <= 0) {
        if (assign) return cudaMemsetAsync(bins, 0, (size_t)nbins * 4, st);
        return cudaSuccess;
    }
    int grid, block;
    if (nbins <= 256) {
        // 16-bit lane counters shared by warp pairs: 4 warps and 34 KB per
        // block, 4 blocks per SM (measured at 2^28: 168 us; one sub-histogram
        // per warp, 3 blocks per SM: 182; the 8-bit form 184; the per-warp
        // form prefetching 2 or 3 chunks ahead 186 / 223; with 6 blocks per SM
        // at <= 80 registers 193 (spills))
        auto kern = pop ? hist256_w16_kernel<true> : hist256_w16_kernel<false>;
        cudaError_t e = set_max_dyn_smem((const void *)kern, kSmemBytes16);
        if (e != cudaSuccess) return e;
        unsigned *acc = (unsigned *)ws;
        // unaligned head keys go to the edge path together with the tail
        int64_t head = (int64_t)(((16 - ((uintptr_t)keys & 15)) & 15) / 4);
        if (head > n) head = n;
        const int64_t n4 = (n - head) / 4;
        const int64_t tail0 = head + 4 * n4;
        const int64_t nchunks = (n4 + kChunk16 - 1) / kChunk16;
        pick_grid(s, (nchunks + kWarps16 - 1) / kWarps16, kBlocksPerSm16, kBlock16, &grid, &block);
        block = kBlock16;
        int64_t edge_head = head;
        if (head > 0 && tail0 < n) {
            // both ends unaligned: count the head into the accumulator first
            hist_big_kernel<<<1, 256, nbins * 4, st>>>(keys, head, (int32_t *)acc, nbins);
            ++*launches;
            edge_head = 0;
        }
        const int32_t *edge = edge_head > 0 ? keys : keys + tail0;
        const int n_edge = (int)(edge_head > 0 ? edge_head : n - tail0);
        kern<<<grid, block, kSmemBytes16, st>>>((const int4 *)(keys + head), n4, edge, n_edge, bins, nbins, acc,
                                                assign ? 1 : 0, pop ? *pop : PeerOp{});
    } else {
        if (assign) {
            cudaError_t e = cudaMemsetAsync(bins, 0, (size_t)nbins * 4, st);
            if (e != cudaSuccess) return e;
        }
        pick_grid(s, (n + 255) / 256, 8, 256, &grid, &block);
        hist_big_kernel<<<grid, block, nbins * 4, st>>>(keys, n, bins, nbins);
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
