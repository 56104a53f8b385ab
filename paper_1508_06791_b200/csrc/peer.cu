// peer.cu -- standalone collective kernels over NVLink peer memory
// (JACC_GRAPH_P2P; protocol and window layout in peer.cuh).  These serve the
// collective tasks that are NOT fused into their producer kernel (the fused
// forms live in histogram.cu, reduce.cu and nbody.cu):
//   allreduce-sum (north_star: "NCCL allreduce of partial sums or bins"),
//   all-gather ("N-body positions by NCCL all-gather over NVLink"),
//   broadcast (SGEMM's replicated B).
// Every rank's kernel both sends (stores into the peers' windows) and
// receives (waits for the peers' data flags), so a task's completion event
// means the result is in place on this rank, like the NCCL call it replaces.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace jacc_k {
namespace {

constexpr int kBlock = 512;

// n small enough for one block: the flag-in-data exchange of peer.cuh.
template <typename T>
__global__ void __launch_bounds__(kBlock) allreduce_small_kernel(PeerCtx c, int slot, int64_t stage_off, T *buf,
                                                                 int64_t n) {
    peer::block_allreduce<T>(c, slot, (size_t)stage_off, buf, n);
}

// Large n, phase 1: every block pushes its slice of buf into row [rank] of
// every rank's staging area (parity e & 1); the last block signals.
template <typename T>
__global__ void __launch_bounds__(kBlock) allreduce_push_kernel(PeerCtx c, int slot, int64_t stage_off,
                                                                const T *buf, int64_t n) {
    const uint64_t e = peer::epoch(c, slot);
    const size_t row = (size_t)n * sizeof(T), half = row * c.world;
    const size_t mine = (size_t)stage_off + (e & 1) * half + (size_t)c.rank * row;
    const size_t per = (row / gridDim.x + 15) & ~(size_t)15;   // 16-byte aligned slices
    const size_t lo = per * blockIdx.x < row ? per * blockIdx.x : row;
    const size_t hi = lo + per < row ? lo + per : row;
    peer::for_each_rank(c, [&](int, char *b) {
        peer::block_copy(b + mine + lo, (const char *)buf + lo, hi - lo, threadIdx.x, blockDim.x);
    });
    if (peer::grid_last(c, slot) && threadIdx.x == 0) peer::publish_data(c, slot, e);
}

// Large n, phase 2 (same stream): wait for every rank, sum rows in rank order.
template <typename T>
__global__ void __launch_bounds__(kBlock) allreduce_sum_kernel(PeerCtx c, int slot, int64_t stage_off, T *buf,
                                                               int64_t n) {
    const uint64_t e = *(volatile uint64_t *)peer::count(c, slot);   // bumped by phase 1
    peer::wait_all_data(c, slot, e);
    __syncthreads();
    const T *rows = (const T *)(c.self + stage_off + (e & 1) * (size_t)n * c.world * sizeof(T));
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        T acc = __ldcg(rows + i);
        for (int q = 1; q < c.world; ++q) acc += __ldcg(rows + (size_t)q * n + i);
        buf[i] = acc;
    }
}

// All-gather (root < 0): rank r's `bytes` of src go to offset dst_off +
// r * bytes of every rank's window (its own included).  Broadcast (root >=
// 0): the root's src goes to offset dst_off of every other rank.  A rank
// that receives first publishes "ready" (its destination is free: the task
// runs after every local reader of it), a sender waits for the receiver's
// ready before storing into it.
__global__ void __launch_bounds__(kBlock) gather_kernel(PeerCtx c, int slot, const char *src, int64_t dst_off,
                                                        int64_t bytes, int root) {
    const uint64_t e = peer::epoch(c, slot);
    const bool receives = root < 0 || c.rank != root;
    if (blockIdx.x == 0 && threadIdx.x == 0 && receives) peer::signal_all(c, peer::kReadyOff, slot, e);
    const size_t per = ((size_t)bytes / gridDim.x + 15) & ~(size_t)15;
    const size_t lo = per * blockIdx.x < (size_t)bytes ? per * blockIdx.x : (size_t)bytes;
    const size_t hi = lo + per < (size_t)bytes ? lo + per : (size_t)bytes;
    if (root < 0 || c.rank == root) {
        const size_t seg = root < 0 ? (size_t)dst_off + (size_t)c.rank * bytes : (size_t)dst_off;
        peer::for_each_rank(c, [&](int q, char *b) {
            if (q == c.rank) {
                if (root < 0) peer::block_copy(b + seg + lo, src + lo, hi - lo, threadIdx.x, blockDim.x);
                return;
            }
            peer::block_wait(c, peer::kReadyOff, slot, q, e);
            peer::block_copy(b + seg + lo, src + lo, hi - lo, threadIdx.x, blockDim.x);
        });
    }
    if (!peer::grid_last(c, slot)) return;
    if (threadIdx.x == 0) peer::publish_data(c, slot, e);
    if (root < 0) peer::wait_all_data(c, slot, e);
    else if (threadIdx.x == 0 && c.rank != root) peer::wait_ge(peer::flag(c.self, peer::kDataOff, slot, root), e);
}

// All ranks: every earlier kernel of this rank's stream has finished (stream
// order) and so have every peer's (each waits for all ranks' flags): after
// this kernel no peer will store into this rank's window again.
__global__ void barrier_kernel(PeerCtx c, int slot) {
    const uint64_t e = peer::epoch(c, slot);
    if (threadIdx.x == 0) peer::publish_data(c, slot, e);
    peer::wait_all_data(c, slot, e);
}

// Halo exchange of row bands (JACC_OP_HALO_EXCHANGE_F32, SURVEY §8(f) f1:
// "shards by row bands with a 2-row halo exchange").  Rank q's band is rows
// [lo_q, lo_q + rows) of one image; ext = [r rows above][band][r rows below].
// A rank does not know its neighbours' band heights, so it does not store
// into their ext directly: it pushes its first r rows into rank q-1's
// staging "from below" and its last r rows into rank q+1's staging "from
// above" (fixed window offsets, same on every rank), publishes, and the
// finish kernel copies its two staging slots into its own ext halos.
// Staging is double-buffered by epoch parity (the allreduce argument: a rank
// cannot write epoch e+2 before every rank signalled e+1, which each does
// only after its finish kernel of epoch e read the staging).
__global__ void __launch_bounds__(kBlock) halo_push_kernel(PeerCtx c, int slot, int64_t stage_off,
                                                           const float *band, float *ext, int64_t rows, int64_t W,
                                                           int r) {
    const uint64_t e = peer::epoch(c, slot);
    const size_t edge = (size_t)r * W * 4, par = (size_t)stage_off + (e & 1) * 2 * edge;
    const size_t body = (size_t)rows * W * 4;
    // this rank's band into the middle of its own ext (grid-wide slices)
    const size_t per = (body / gridDim.x + 15) & ~(size_t)15;
    const size_t lo = per * blockIdx.x < body ? per * blockIdx.x : body;
    const size_t hi = lo + per < body ? lo + per : body;
    peer::block_copy((char *)ext + edge + lo, (const char *)band + lo, hi - lo, threadIdx.x, blockDim.x);
    // edges to the neighbours' staging (block 0 only: 2 x r rows)
    if (blockIdx.x == 0) {
        peer::for_each_rank(c, [&](int q, char *b) {
            if (q == c.rank - 1)        // rank above receives our first r rows as "from below"
                peer::block_copy(b + par + edge, (const char *)band, edge, threadIdx.x, blockDim.x);
            else if (q == c.rank + 1)   // rank below receives our last r rows as "from above"
                peer::block_copy(b + par, (const char *)band + body - edge, edge, threadIdx.x, blockDim.x);
        });
    }
    if (peer::grid_last(c, slot) && threadIdx.x == 0) peer::publish_data(c, slot, e);
}

__global__ void __launch_bounds__(kBlock) halo_finish_kernel(PeerCtx c, int slot, int64_t stage_off, float *ext,
                                                             int64_t rows, int64_t W, int r) {
    const uint64_t e = *(volatile uint64_t *)peer::count(c, slot);   // bumped by the push kernel
    peer::wait_all_data(c, slot, e);
    __syncthreads();
    const size_t edge = (size_t)r * W * 4, par = (size_t)stage_off + (e & 1) * 2 * edge;
    const int64_t n = (int64_t)r * W;
    float *top = ext, *bot = ext + (size_t)(r + rows) * W;
    const float *from_above = (const float *)(c.self + par), *from_below = (const float *)(c.self + par + edge);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        top[i] = c.rank > 0 ? __ldcg(from_above + i) : 0.f;
        bot[i] = c.rank < c.world - 1 ? __ldcg(from_below + i) : 0.f;
    }
}

// One rank (world 1, or the NCCL path's local part): band into the middle,
// zeros for the halos past the image.
__global__ void __launch_bounds__(kBlock) halo_local_kernel(const float *band, float *ext, int64_t rows, int64_t W,
                                                            int r, int top_zero, int bottom_zero) {
    const int64_t n = (int64_t)rows * W, h = (int64_t)r * W;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n + 2 * h;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < h) {
            if (top_zero) ext[i] = 0.f;
        } else if (i < h + n) {
            ext[i] = __ldg(band + (i - h));
        } else if (bottom_zero) {
            ext[i] = 0.f;
        }
    }
}

int copy_grid(int64_t bytes) {
    // ~64 KiB per block, at most 32 blocks (a few SMs: the copy is NVLink-bound)
    int64_t g = (bytes + (64 << 10) - 1) / (64 << 10);
    return (int)(g < 1 ? 1 : g > 32 ? 32 : g);
}

}  // namespace

size_t peer_allreduce_stage_bytes(int64_t n, int, int world) { return peer::allreduce_stage_bytes(n, world); }

cudaError_t peer_allreduce(const PeerOp &op, void *buf, int64_t n, bool is_int, cudaStream_t st, int *launches) {
    const int esz = 4;
    if (n <= peer::kSmallN) {
        if (is_int)
            allreduce_small_kernel<int><<<1, kBlock, 0, st>>>(op.ctx, op.slot, op.off, (int *)buf, n);
        else
            allreduce_small_kernel<float><<<1, kBlock, 0, st>>>(op.ctx, op.slot, op.off, (float *)buf, n);
        ++*launches;
        return cudaGetLastError();
    }
    const int g = copy_grid(n * esz);
    if (is_int) {
        allreduce_push_kernel<int><<<g, kBlock, 0, st>>>(op.ctx, op.slot, op.off, (const int *)buf, n);
        allreduce_sum_kernel<int><<<g, kBlock, 0, st>>>(op.ctx, op.slot, op.off, (int *)buf, n);
    } else {
        allreduce_push_kernel<float><<<g, kBlock, 0, st>>>(op.ctx, op.slot, op.off, (const float *)buf, n);
        allreduce_sum_kernel<float><<<g, kBlock, 0, st>>>(op.ctx, op.slot, op.off, (float *)buf, n);
    }
    *launches += 2;
    return cudaGetLastError();
}

size_t peer_halo_stage_bytes(int64_t W, int radius) { return 2 * 2 * (size_t)radius * W * 4; }

cudaError_t peer_halo(const PeerOp &op, const float *band, float *ext, int64_t rows, int64_t W, int radius,
                      cudaStream_t st, int *launches) {
    const int64_t bytes = rows * W * 4;
    const int g = (int)std::min<int64_t>(148, std::max<int64_t>(1, bytes / (256 << 10)));
    halo_push_kernel<<<g, kBlock, 0, st>>>(op.ctx, op.slot, op.off, band, ext, rows, W, radius);
    const int g2 = (int)std::min<int64_t>(32, std::max<int64_t>(1, (int64_t)radius * W / 8192));
    halo_finish_kernel<<<g2, kBlock, 0, st>>>(op.ctx, op.slot, op.off, ext, rows, W, radius);
    *launches += 2;
    return cudaGetLastError();
}

cudaError_t halo_local(const float *band, float *ext, int64_t rows, int64_t W, int radius, bool top_zero,
                       bool bottom_zero, cudaStream_t st, int *launches) {
    const int64_t n = (rows + 2 * radius) * W;
    const int g = (int)std::min<int64_t>(148 * 8, std::max<int64_t>(1, (n + kBlock * 4 - 1) / (kBlock * 4)));
    halo_local_kernel<<<g, kBlock, 0, st>>>(band, ext, rows, W, radius, top_zero, bottom_zero);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t peer_allgather(const PeerOp &op, const void *send, int64_t bytes, cudaStream_t st, int *launches) {
    gather_kernel<<<copy_grid(bytes), kBlock, 0, st>>>(op.ctx, op.slot, (const char *)send, op.off, bytes, -1);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t peer_broadcast(const PeerOp &op, int root, int64_t bytes, cudaStream_t st, int *launches) {
    const char *src = op.ctx.self + op.off;
    gather_kernel<<<copy_grid(bytes), kBlock, 0, st>>>(op.ctx, op.slot, src, op.off, bytes, root);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k

namespace jacc_k {
cudaError_t peer_barrier(const PeerCtx &c, int slot, cudaStream_t st) {
    barrier_kernel<<<1, 32, 0, st>>>(c, slot);
    return cudaGetLastError();
}
}  // namespace jacc_k
