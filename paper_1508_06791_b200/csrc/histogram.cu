// histogram.cu -- Histogram (§4.2): "frequency counts for
// ... values, placing the results into 256 distinct bins"; the bins are an
// @Atomic(op=ADD) output (Table 1) updated "using shared memory
// atomic operations" and auto-zeroed.
//
// bins[k] += #{i : keys[i] == k} for 0 <= k < nbins; other keys are ignored
// (reading R11).  Integer counts: bit-exact by construction.
//
// sm_100a design (nbins <= 256), sized so the HBM read of 4 B/key binds:
//   * privatisation at the finest grain -- every LANE owns a private 8-bit
//     sub-histogram in shared memory, laid out word (bin/4)*32 + lane, byte
//     bin%4.  A lane's word always sits in bank `lane`, so the 32 updates of
//     a warp never conflict, for ANY key distribution (uniform or all-equal);
//     the update is a shared-memory atomic add whose result is unused (no
//     dependency chain between a lane's keys).
//   * keys stream in as 128-bit loads, 4 int4 per lane per chunk, with the
//     next chunk prefetched into registers while the current one is counted.
//   * before an 8-bit counter can overflow (<= 240 keys per lane) the warp
//     folds its sub-histograms into per-lane 32-bit register totals (lane l
//     owns bins 8l..8l+7; column reads are rotated so they stay
//     conflict-free) and clears them;
//   * at the end the warps' totals are combined with shared-memory atomics
//     into one block histogram, merged ONCE per block into global memory
//     with 256 atomicAdds.
// nbins in (256, 4096]: a plain shared-memory-atomics block histogram.
//
// JACC_GRAPH_P2P fusion (reading R23): when the graph's next task is the
// allreduce of these bins, the same kernel finishes it -- the last block to
// merge (grid ticket) pushes the local bins into every rank's window over
// NVLink, waits for the other ranks' rows and sums them in rank order
// (peer.cuh block_allreduce): one launch instead of histogram + NCCL.
#include "common.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace jacc_k {
namespace {

constexpr int kWarps = 8;                 // 256 threads
constexpr int kBlock = kWarps * 32;
constexpr int kU = 4;                     // int4 per lane per chunk (16 keys); 8 measured slower (0.196 vs 0.186 ms at 2^28)
constexpr int kChunk = 32 * kU;           // int4 per warp chunk
constexpr int kFlushChunks = 15;          // 15 * 16 = 240 keys <= 255 per lane
constexpr int kSubWords = 65 * 32;        // 256 bins * 32 lanes / 4 per word + 1 dummy group
constexpr int kSmemBytes = kWarps * kSubWords * 4 + 256 * 4;

// Fold the warp's 8-bit sub-histograms into lane l's totals of bins 8l..8l+7.
__device__ __forceinline__ void flush(unsigned *sub, unsigned lane, unsigned tot[8]) {
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const unsigned g = 2 * lane + h;               // word group: bins 4g..4g+3
        unsigned even = 0, odd = 0;                    // 16-bit lanes: bins 4g+{0,2} / 4g+{1,3}
#pragma unroll 8
        for (unsigned c = 0; c < 32; ++c) {
            const unsigned v = sub[g * 32 + ((c + lane) & 31)];
            even += v & 0x00FF00FFu;
            odd += (v >> 8) & 0x00FF00FFu;
        }
        tot[4 * h + 0] += even & 0xFFFFu;
        tot[4 * h + 1] += odd & 0xFFFFu;
        tot[4 * h + 2] += even >> 16;
        tot[4 * h + 3] += odd >> 16;
    }
    __syncwarp();
#pragma unroll 8
    for (int g = 0; g < 64; ++g) sub[g * 32 + lane] = 0u;
    __syncwarp();
}

// One key, branch-free: a key outside [0, nbins) is clamped to bin `nbins`
// (<= 256), a bin that is never merged into the output (bin 256 = dummy group
// 64).  The lane's byte counter of bin kk lives in its word (kk/4)*32 + lane
// (bank `lane`: a warp's 32 updates never conflict) at byte kk%4, and is
// bumped with a shared-memory atomic add of 1 << 8 (kk%4) whose result is not
// used -- one smem op per key and no load -> add -> store dependency chain.
// (Measured: plain byte LDS/IADD/STS 193 us, with 2 or 4 updates per lane in
// flight 200 / 230 us, this 188 us at 2^28 keys.)
__device__ __forceinline__ void count_key(unsigned *sub_lane_w, int k, unsigned nbins) {
    const unsigned kk = min((unsigned)k, nbins);
    atomicAdd(sub_lane_w + ((kk >> 2) << 5), 1u << ((kk & 3u) << 3));
}

template <bool kPeer>
__global__ void __launch_bounds__(kBlock) hist256_kernel(const int4 *__restrict__ keys4, int64_t n4,
                                                         const int32_t *__restrict__ edge, int n_edge,
                                                         int32_t *__restrict__ bins, int nbins, PeerOp pop) {
    extern __shared__ unsigned smem[];
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned *sub = smem + warp * kSubWords;
    unsigned *blockh = smem + kWarps * kSubWords;
    for (int g = 0; g < 65; ++g) sub[g * 32 + lane] = 0u;
    if (threadIdx.x < 256) blockh[threadIdx.x] = 0u;
    __syncthreads();

    unsigned tot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int64_t nwarps = (int64_t)gridDim.x * kWarps;
    int64_t c = (int64_t)blockIdx.x * kWarps + warp;
    const int64_t nchunks = (n4 + kChunk - 1) / kChunk;
    int since_flush = 0;
    int4 cur[kU], nxt[kU];
    auto load = [&](int64_t ch, int4 *dst) {
        if ((ch + 1) * kChunk <= n4) {   // interior chunk: unconditional 128-bit loads
#pragma unroll
            for (int u = 0; u < kU; ++u) dst[u] = ld_stream(keys4 + ch * kChunk + u * 32 + lane);
        } else {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int64_t idx = ch * kChunk + u * 32 + lane;
                dst[u] = (ch < nchunks && idx < n4) ? ld_stream(keys4 + idx) : make_int4(-1, -1, -1, -1);
            }
        }
    };
    if (c < nchunks) load(c, cur);
    for (; c < nchunks; c += nwarps) {
        load(c + nwarps, nxt);   // prefetch the next chunk of this warp
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            count_key(sub + lane, cur[u].x, nbins);
            count_key(sub + lane, cur[u].y, nbins);
            count_key(sub + lane, cur[u].z, nbins);
            count_key(sub + lane, cur[u].w, nbins);
        }
        if (++since_flush == kFlushChunks) {
            flush(sub, lane, tot);
            since_flush = 0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) cur[u] = nxt[u];
    }
    // keys outside the 128-bit body (unaligned head / < 4 tail): block 0
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < n_edge; i += kBlock) {
            const int k = edge[i];
            if ((unsigned)k < (unsigned)nbins) atomicAdd(&blockh[k], 1u);
        }
    }
    flush(sub, lane, tot);
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (tot[j]) atomicAdd(&blockh[8 * lane + j], tot[j]);
    __syncthreads();
    // merged once per block into the global @Atomic bins
    if (threadIdx.x < nbins && blockh[threadIdx.x]) atomicAdd(&bins[threadIdx.x], (int)blockh[threadIdx.x]);
    if (kPeer && peer::grid_last(pop.ctx, pop.slot))   // every block's bins are in: allreduce them
        peer::block_allreduce<int>(pop.ctx, pop.slot, (size_t)pop.off, bins, nbins);
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

size_t histogram_ws_bytes(int64_t, int) { return 0; }

cudaError_t histogram_i32(const int32_t *keys, int64_t n, int32_t *bins, int nbins, void *, const jacc_schedule_t *s,
                          cudaStream_t st, int *launches, const PeerOp *pop) {
    if (pop && (n <= 0 || nbins > 256)) return cudaErrorInvalidValue;   // the runtime only fuses these
    if (n <= 0) return cudaSuccess;
    int grid, block;
    if (nbins <= 256) {
        auto kern = pop ? hist256_kernel<true> : hist256_kernel<false>;
        cudaError_t e = set_max_dyn_smem((const void *)kern, kSmemBytes);
        if (e != cudaSuccess) return e;
        // unaligned head keys go to the edge path together with the tail
        int64_t head = (int64_t)(((16 - ((uintptr_t)keys & 15)) & 15) / 4);
        if (head > n) head = n;
        const int64_t n4 = (n - head) / 4;
        const int64_t tail0 = head + 4 * n4;
        const int64_t nchunks = (n4 + kChunk * 1 - 1) / kChunk;
        // 3 x 66 KB blocks per SM; the edge keys: [0, head) and [tail0, n)
        pick_grid(s, (nchunks + kWarps - 1) / kWarps, 3, kBlock, &grid, &block);
        block = kBlock;
        int64_t edge_head = head;
        if (head > 0 && tail0 < n) {
            // both ends unaligned: count the head with the small generic kernel
            hist_big_kernel<<<1, 256, nbins * 4, st>>>(keys, head, bins, nbins);
            ++*launches;
            edge_head = 0;
        }
        const int32_t *edge = edge_head > 0 ? keys : keys + tail0;
        const int n_edge = (int)(edge_head > 0 ? edge_head : n - tail0);
        kern<<<grid, block, kSmemBytes, st>>>((const int4 *)(keys + head), n4, edge, n_edge, bins, nbins,
                                              pop ? *pop : PeerOp{});
    } else {
        pick_grid(s, (n + 255) / 256, 8, 256, &grid, &block);
        hist_big_kernel<<<grid, block, nbins * 4, st>>>(keys, n, bins, nbins);
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
