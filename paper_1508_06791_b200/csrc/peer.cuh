// peer.cuh -- collectives over NVLink peer memory (JACC_GRAPH_P2P).
//
// The north_star's exchange steps -- allreduce of partial bins / sums,
// all-gather of N-body positions, broadcast (reading R17: SPMD, one process
// per GPU, collectives are graph tasks) -- run here as plain loads and stores
// into the other GPUs' memory, fused into the kernel that produces the data
// where one does (histogram -> allreduce, reduce -> allreduce, N-body step ->
// all-gather), instead of a separate NCCL call.
//
// Symmetric window.  Every rank cudaMalloc's one window of the same size,
// exports its CUDA IPC handle, and maps every other rank's window
// (jacc_peer_init / jacc_peer_connect).  Offsets inside the window are the
// same on every rank (SPMD: identical graphs and jacc_peer_alloc calls), so
// "offset o in rank q's window" is base[q] + o.
//
// Window header (per rank):
//   data [kSlots][kMaxPeers]  u64  written by rank src: "my data for slot s,
//                                   epoch e, is in your window"
//   ready[kSlots][kMaxPeers]  u64  written by rank src: "my receive buffer of
//                                   slot s is free for epoch e"
//   count[kSlots]             u64  local: epochs of slot s completed here
//   ticket[kSlots]            u32  local: grid-completion ticket
// Every collective task has a slot (its index among the graph's collective
// tasks).  Epoch e of slot s = the e-th execution of that task; all ranks
// run the same tasks, so e agrees across ranks without any host input (and
// a captured CUDA graph replays correctly).  A flag only grows, so it never
// needs resetting; a waiter checks flag >= e.
//
// Ordering: data stores (st.global to the mapped peer address), then
// __syncthreads + fence.sc.sys by one thread, then the grid ticket; the last
// block fences again and publishes the flag with st.release.sys; the waiter
// polls with ld.acquire.sys and its block reads the data after a barrier,
// through L2 (ld.cg / cp.async.cg), never the non-coherent path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace jacc_k {
namespace peer {

constexpr int kMaxPeers = JACC_PEER_MAX;   // one NVLink/NVSwitch domain (8 GPUs per box)
constexpr int kSlots = 1024;
constexpr size_t kDataOff = 0;
constexpr size_t kReadyOff = kDataOff + sizeof(uint64_t) * kSlots * kMaxPeers;
constexpr size_t kCountOff = kReadyOff + sizeof(uint64_t) * kSlots * kMaxPeers;
constexpr size_t kTicketOff = kCountOff + sizeof(uint64_t) * kSlots;
constexpr size_t kHeaderBytes = 256 * 1024;   // heap starts here
static_assert(kTicketOff + sizeof(unsigned) * kSlots <= kHeaderBytes, "peer header");

// spin limit: a peer that has not arrived after this long is a protocol or
// SPMD error (different graphs on different ranks); the kernel traps and the
// graph's sync reports JACC_ERR_CUDA instead of hanging the GPU.
constexpr unsigned long long kTimeoutNs = 30ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint64_t *flag(char *base, size_t off, int slot, int src) {
    return (uint64_t *)(base + off) + (size_t)slot * kMaxPeers + src;
}
__device__ __forceinline__ uint64_t *count(const PeerCtx &c, int slot) {
    return (uint64_t *)(c.base[c.rank] + kCountOff) + slot;
}
__device__ __forceinline__ unsigned *ticket(const PeerCtx &c, int slot) {
    return (unsigned *)(c.base[c.rank] + kTicketOff) + slot;
}

__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin (one thread) until *p >= e.
__device__ __forceinline__ void wait_ge(const uint64_t *p, uint64_t e) {
    if (ld_acquire_sys(p) >= e) return;
    const uint64_t t0 = globaltimer();
    for (unsigned it = 1;; ++it) {
        __nanosleep(100);
        if (ld_acquire_sys(p) >= e) return;
        if ((it & 1023u) == 0 && globaltimer() - t0 > kTimeoutNs) __trap();
    }
}

// Epoch of the current execution of `slot` (all threads may call it before
// the slot's last block bumps the count).
__device__ __forceinline__ uint64_t epoch(const PeerCtx &c, int slot) {
    return *(volatile uint64_t *)count(c, slot) + 1;
}

// One thread: publish flag (data or ready) of `slot` = e to every rank.
__device__ __forceinline__ void signal_all(const PeerCtx &c, size_t off, int slot, uint64_t e) {
    for (int q = 0; q < c.world; ++q) st_release_sys(flag(c.base[q], off, slot, c.rank), e);
}

// Whole block: wait until rank q's flag (in OUR header) reached e.
__device__ __forceinline__ void block_wait(const PeerCtx &c, size_t off, int slot, int q, uint64_t e) {
    if (threadIdx.x == 0) wait_ge(flag(c.base[c.rank], off, slot, q), e);
    __syncthreads();
}

// Whole block: copy `bytes` (multiple of 4) from local src to dst (any rank's
// memory), 16-byte vectors when both are 16-byte aligned.
__device__ __forceinline__ void block_copy(char *dst, const char *src, size_t bytes, size_t tid, size_t nthr) {
    if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
        const size_t n16 = bytes / 16;
        for (size_t i = tid; i < n16; i += nthr) ((int4 *)dst)[i] = __ldcg((const int4 *)src + i);
        for (size_t i = n16 * 16 + tid * 4; i < bytes; i += nthr * 4)
            *(int *)(dst + i) = __ldcg((const int *)(src + i));
    } else {
        for (size_t i = tid * 4; i < bytes; i += nthr * 4) *(int *)(dst + i) = __ldcg((const int *)(src + i));
    }
}

// Grid completion: every block calls this after its stores (to any rank);
// returns true in exactly one block (the last), in which every thread may
// then rely on all blocks' stores being visible system-wide.
__device__ __forceinline__ bool grid_last(const PeerCtx &c, int slot) {
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        s_last = atomicAdd(ticket(c, slot), 1u) == gridDim.x - 1;
        if (s_last) {
            *ticket(c, slot) = 0u;   // re-arm (stream-ordered before the next launch)
            __threadfence_system();
        }
    }
    __syncthreads();
    return s_last;
}

// Whole block, ONE block of the grid: allreduce-sum of buf[0..n) over all
// ranks.  Pushes buf into every rank's staging row [rank] (double-buffered by
// epoch parity: a fast rank's next epoch never overwrites rows a slow rank is
// still summing -- it cannot start epoch e+2 before every rank signalled e+1,
// which each does only after summing e), signals, waits for every rank and
// sums the rows in rank order (deterministic; bit-exact for integers).
template <typename T>
__device__ __forceinline__ void block_allreduce(const PeerCtx &c, int slot, size_t stage_off, T *buf, int64_t n) {
    const uint64_t e = epoch(c, slot);
    const size_t row = (size_t)n * sizeof(T);
    const size_t half = row * c.world;
    const size_t mine = stage_off + (e & 1) * half + (size_t)c.rank * row;
    __syncthreads();
    for (int q = 0; q < c.world; ++q)
        block_copy(c.base[q] + mine, (const char *)buf, row, threadIdx.x, blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        signal_all(c, kDataOff, slot, e);
        *count(c, slot) = e;
    }
    if (threadIdx.x < (unsigned)c.world) wait_ge(flag(c.base[c.rank], kDataOff, slot, threadIdx.x), e);
    __syncthreads();
    const T *rows = (const T *)(c.base[c.rank] + stage_off + (e & 1) * half);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        T acc = __ldcg(rows + i);
        for (int q = 1; q < c.world; ++q) acc += __ldcg(rows + (size_t)q * n + i);
        buf[i] = acc;
    }
}

}  // namespace peer
}  // namespace jacc_k
