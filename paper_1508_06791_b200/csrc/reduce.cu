// reduce.cu -- Reduction (§2.1.2; §4.2):
// out[0] += sum_i x[i].
//
// The paper's Jacc kernel assigns every partial to an @Atomic(op=ADD) field,
// "effectively turning the assignment into: result += sum", auto-
// zeroed (the runtime's MEMSET0 action), and reduces atomic
// contention by launching fewer threads.  On sm_100a the same
// result is reached without float atomics (reading R14):
//   1. 128-bit streaming loads, 4 independent fp32 accumulators per thread;
//   2. warp shuffle-xor tree, then a block tree through shared memory;
//   3. SINGLE-PASS cross-block finish: each block stores its partial, bumps
//      an atomic ticket; the last block to arrive sums the partials in block
//      order and adds the total to out[0], then re-arms the ticket.
// For a given n the grid is fixed, so the result is bitwise reproducible.
// HBM-bound: 4 algorithmic bytes per element.
//
// JACC_GRAPH_P2P fusion (reading R23): when the next task is the allreduce
// of out, the last block also completes it over NVLink peer memory (push the
// local total to every rank, wait, sum the ranks' totals in rank order).
#include "common.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace jacc_k {
namespace {

constexpr int kBlock = 512;
constexpr int kPerSm = 4;           // 4 x 512 threads = 2048 resident per SM
constexpr int kMaxGrid = 148 * 8;   // workspace sized for any B200 grid

__device__ __forceinline__ float block_sum(float v, float *sh) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    v = (threadIdx.x < (blockDim.x >> 5)) ? sh[lane] : 0.f;
    if (warp == 0) v = warp_sum(v);
    return v;   // valid in thread 0
}

// kFused (the runtime's "merge" of vadd -> reduce): the element
// value is a[i] + b[i] (one fp32 add, exactly the vadd kernel's), stored to
// c and summed in the very same order as reduce_kernel<false> on c -- so the
// merged pair produces bit-identical c and s in one pass over a and b.
template <bool kFused, bool kPeer>
__global__ void __launch_bounds__(kBlock, 2) reduce_kernel(const float *__restrict__ x, const float *__restrict__ xb,
                                                        float *__restrict__ xc, int64_t n, int64_t head,
                                                        float *__restrict__ out, float *__restrict__ partials,
                                                        unsigned *__restrict__ ticket, int assign, PeerOp pop) {
    __shared__ float sh[32];
    __shared__ bool last;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
    // unaligned head (< 4 scalars), then 128-bit body, then tail (< 4 scalars)
    auto elem = [&](int64_t j) -> float {
        if (!kFused) return x[j];
        const float v = x[j] + xb[j];
        xc[j] = v;
        return v;
    };
    auto vec = [&](int64_t j) -> float4 {   // j indexes float4 from x + head
        float4 u = ld_stream((const float4 *)(x + head) + j);
        if (kFused) {
            const float4 w = ld_stream((const float4 *)(xb + head) + j);
            u = make_float4(u.x + w.x, u.y + w.y, u.z + w.z, u.w + w.w);
            st_stream((float4 *)(xc + head) + j, u);
        }
        return u;
    };
    if (tid < head) a0 += elem(tid);
    const int64_t n4 = (n - head) / 4;
    int64_t i = tid;
    // 4 vectors in flight per thread (2 left the read stream at ~5.76 TB/s)
    for (; i + 3 * stride < n4; i += 4 * stride) {
        const float4 u = vec(i), v = vec(i + stride), w = vec(i + 2 * stride), z = vec(i + 3 * stride);
        a0 += u.x; a1 += u.y; a2 += u.z; a3 += u.w;
        a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w;
        a0 += w.x; a1 += w.y; a2 += w.z; a3 += w.w;
        a0 += z.x; a1 += z.y; a2 += z.z; a3 += z.w;
    }
    if (i < n4) {   // the remainder (< 4 vectors): loads issued together, added in index order
        const bool h1 = i + stride < n4, h2 = i + 2 * stride < n4;
        const float4 u = vec(i);
        const float4 v = h1 ? vec(i + stride) : make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 w = h2 ? vec(i + 2 * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
        a0 += u.x; a1 += u.y; a2 += u.z; a3 += u.w;
        if (h1) { a0 += v.x; a1 += v.y; a2 += v.z; a3 += v.w; }
        if (h2) { a0 += w.x; a1 += w.y; a2 += w.z; a3 += w.w; }
    }
    const int64_t t0 = head + 4 * n4;
    if (tid < n - t0) a1 += elem(t0 + tid);
    float s = block_sum((a0 + a1) + (a2 + a3), sh);
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = s;
        __threadfence();
        last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    float p = 0.f;
    for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) p += __ldcg(partials + b);
    p = block_sum(p, sh);
    if (threadIdx.x == 0) {
        // @Atomic ADD semantics: result += sum; a W output is
        // auto-zeroed, i.e. result = 0 + sum -- stored directly
        out[0] = assign ? 0.f + p : out[0] + p;
        *ticket = 0u;      // re-arm for the next launch (stream-ordered)
    }
    if (kPeer) peer::block_allreduce<float>(pop.ctx, pop.slot, (size_t)pop.off, out, 1);
}

}  // namespace

size_t reduce_ws_bytes(int64_t) { return sizeof(float) * kMaxGrid + 128; }

namespace {
void reduce_grid(int64_t n, const jacc_schedule_t *s, int *grid, int *block) {
    // one resident wave: with <= 64 registers (launch bounds) 2 blocks of
    // 512 fit per SM, not kPerSm -- a grid of 4 per SM ran as two waves (the
    // second starting as the first drained).  The same grid for every
    // instantiation: the merged vadd+reduce must sum in the plain order.
    static const int occ = blocks_per_sm((const void *)reduce_kernel<false, false>, kBlock, 0);
    pick_grid(s, (n / 4 + kBlock * 2 - 1) / (kBlock * 2), occ < kPerSm ? occ : kPerSm, kBlock, grid, block);
    *block = kBlock;   // the block tree assumes kBlock threads
    if (*grid > kMaxGrid) *grid = kMaxGrid;
}
}  // namespace

cudaError_t reduce_sum_f32(const float *x, int64_t n, float *out, void *ws, const jacc_schedule_t *s,
                           cudaStream_t st, int *launches, bool assign, const PeerOp *pop) {
    int grid, block;
    const int64_t head = (int64_t)(((16 - ((uintptr_t)x & 15)) & 15) / 4) < n
                             ? (int64_t)(((16 - ((uintptr_t)x & 15)) & 15) / 4)
                             : n;
    reduce_grid(n, s, &grid, &block);
    float *partials = (float *)ws;
    unsigned *ticket = (unsigned *)((char *)ws + sizeof(float) * kMaxGrid);
    if (pop)
        reduce_kernel<false, true><<<grid, block, 0, st>>>(x, nullptr, nullptr, n, head, out, partials, ticket,
                                                           assign, *pop);
    else
        reduce_kernel<false, false><<<grid, block, 0, st>>>(x, nullptr, nullptr, n, head, out, partials, ticket,
                                                            assign, PeerOp{});
    ++*launches;
    return cudaGetLastError();
}

bool vadd_reduce_fusable(const float *a, const float *b, const float *c) {
    return aligned16(a) && aligned16(b) && aligned16(c);
}

// c = a + b and out[0] += sum(c) in one pass (requires vadd_reduce_fusable).
cudaError_t vadd_reduce_f32(const float *a, const float *b, float *c, int64_t n, float *out, void *ws,
                            const jacc_schedule_t *s_reduce, cudaStream_t st, int *launches, bool assign,
                            const PeerOp *pop) {
    int grid, block;
    reduce_grid(n, s_reduce, &grid, &block);
    float *partials = (float *)ws;
    unsigned *ticket = (unsigned *)((char *)ws + sizeof(float) * kMaxGrid);
    if (pop)
        reduce_kernel<true, true><<<grid, block, 0, st>>>(a, b, c, n, 0, out, partials, ticket, assign, *pop);
    else
        reduce_kernel<true, false><<<grid, block, 0, st>>>(a, b, c, n, 0, out, partials, ticket, assign, PeerOp{});
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
