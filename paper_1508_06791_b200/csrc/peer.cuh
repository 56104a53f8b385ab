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
// __syncthreads + fence.acq_rel.sys by one thread, then the grid ticket; the
// last block fences again and publishes the flag; the waiter polls with
// relaxed system-scope loads, fences (acquire) once the flag matches, and
// its block reads the data through L2 (ld.cg), never the non-coherent path.
// Small allreduces skip all of this: their values carry the epoch inside
// each 8-byte word (block_allreduce, "LL" = low latency).
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
    return (uint64_t *)(c.self + kCountOff) + slot;
}
__device__ __forceinline__ unsigned *ticket(const PeerCtx &c, int slot) {
    return (unsigned *)(c.self + kTicketOff) + slot;
}

// f(q, base_q) for every rank q.  The loop is unrolled over the constant
// bound so base[] is only ever indexed by constants: a runtime index into a
// by-value kernel parameter array makes the compiler copy the whole struct
// to local memory (a stack frame and local loads for every access).
template <typename F>
__device__ __forceinline__ void for_each_rank(const PeerCtx &c, F &&f) {
#pragma unroll
    for (int q = 0; q < kMaxPeers; ++q)
        if (q < c.world) f(q, c.base[q]);
}

__device__ __forceinline__ void st_release_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Polling load: relaxed (an acquire load invalidates L1 on every poll);
// the waiter issues one acquire fence after the wait succeeds.
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Spin (one thread) until pred(*p) holds; then acquire (kAcquire: later
// loads of OTHER data must see what the flag's writer stored before it).
template <bool kAcquire = true, typename Pred>
__device__ __forceinline__ uint64_t spin_until(const uint64_t *p, Pred pred) {
    uint64_t v = ld_relaxed_sys(p);
    if (!pred(v)) {
        const uint64_t t0 = globaltimer();
        for (unsigned it = 1;; ++it) {
            __nanosleep(32);
            v = ld_relaxed_sys(p);
            if (pred(v)) break;
            if ((it & 1023u) == 0 && globaltimer() - t0 > kTimeoutNs) __trap();
        }
    }
    if (kAcquire) fence_acq_rel_sys();
    return v;
}

// Spin (one thread) until *p >= e.
__device__ __forceinline__ void wait_ge(const uint64_t *p, uint64_t e) {
    spin_until(p, [e](uint64_t v) { return v >= e; });
}

// Epoch of the current execution of `slot` (all threads may call it before
// the slot's last block bumps the count).
__device__ __forceinline__ uint64_t epoch(const PeerCtx &c, int slot) {
    return *(volatile uint64_t *)count(c, slot) + 1;
}

// One thread: publish flag (data or ready) of `slot` = e to every rank.
__device__ __forceinline__ void signal_all(const PeerCtx &c, size_t off, int slot, uint64_t e) {
    for_each_rank(c, [&](int, char *b) { st_release_sys(flag(b, off, slot, c.rank), e); });
}

// Whole block: wait until rank q's flag (in OUR header) reached e.
__device__ __forceinline__ void block_wait(const PeerCtx &c, size_t off, int slot, int q, uint64_t e) {
    if (threadIdx.x == 0) wait_ge(flag(c.self, off, slot, q), e);
    __syncthreads();
}

// Threads 0 .. world-1 of a block: wait for every rank's data flag >= e.
__device__ __forceinline__ void wait_all_data(const PeerCtx &c, int slot, uint64_t e) {
    if (threadIdx.x < (unsigned)c.world) wait_ge(flag(c.self, kDataOff, slot, threadIdx.x), e);
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

// Grid completion: every block calls this after its stores; returns true in
// exactly one block (the last), in which every thread may then rely on all
// blocks' stores being visible.  The fence before the ticket is GPU-scope
// even when the blocks stored into PEER memory: every block synchronizes
// with the last block at GPU scope (release fence + ticket atomic, atomic +
// acquire fence: all on this GPU), and the last block's system-scope fence
// in publish_data synchronizes with the peers' acquire -- causality order is
// transitive across the two synchronizations (PTX memory model), so a peer
// that sees the flag sees every block's stores.  (A system-scope fence per
// block measured ~3 us slower on the N-body step.)
__device__ __forceinline__ bool grid_last(const PeerCtx &c, int slot) {
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        s_last = atomicAdd(ticket(c, slot), 1u) == gridDim.x - 1;
        if (s_last) {
            *ticket(c, slot) = 0u;   // re-arm (stream-ordered before the next launch)
            fence_acq_rel_gpu();     // acquire side of the ticket
        }
    }
    __syncthreads();
    return s_last;
}

// Publish "data of epoch e" to every rank (one thread, after a block barrier
// that follows the block's -- and, via grid_last, the grid's -- stores).
__device__ __forceinline__ void publish_data(const PeerCtx &c, int slot, uint64_t e) {
    fence_acq_rel_sys();
    for_each_rank(c, [&](int, char *b) { st_relaxed_sys(flag(b, kDataOff, slot, c.rank), e); });
    *count(c, slot) = e;
}

template <typename T> __device__ __forceinline__ uint32_t to_bits(T v);
template <> __device__ __forceinline__ uint32_t to_bits<int>(int v) { return (uint32_t)v; }
template <> __device__ __forceinline__ uint32_t to_bits<float>(float v) { return __float_as_uint(v); }
template <typename T> __device__ __forceinline__ T from_bits(uint32_t v);
template <> __device__ __forceinline__ int from_bits<int>(uint32_t v) { return (int)v; }
template <> __device__ __forceinline__ float from_bits<float>(uint32_t v) { return __uint_as_float(v); }

// Allreduces of up to kSmallN elements use the one-block flag-in-data form
// below (8-byte words); larger ones the two-kernel form (4-byte rows + flags).
constexpr int64_t kSmallN = 8192;

// Bytes of staging one allreduce slot needs: 2 epoch parities x world rows.
__host__ __device__ inline size_t allreduce_stage_bytes(int64_t n, int world) {
    return 2 * (size_t)n * (n <= kSmallN ? 8 : 4) * world;
}

// Whole block, ONE block of the grid: allreduce-sum of buf[0..n) over all
// ranks with the flag-in-data ("LL") protocol -- every 4-byte value travels
// in one 8-byte word {value, epoch} stored with a single 64-bit store into
// row [rank] of every rank's staging area, and the receiver polls the words
// themselves until their epoch tag matches: no fence, no separate flag, one
// NVLink write + read of latency.  Rows are double-buffered by epoch parity:
// a rank cannot write epoch e+2 before every rank has written e+1, which each
// does only after it finished reading e.  Rows are summed in rank order
// (deterministic; bit-exact for integers).
template <typename T>
__device__ __forceinline__ void block_allreduce(const PeerCtx &c, int slot, size_t stage_off, T *buf, int64_t n) {
    __shared__ uint64_t s_e;
    __syncthreads();                       // buf is final (written by this block / seen via grid_last)
    if (threadIdx.x == 0) s_e = epoch(c, slot);
    __syncthreads();
    const uint64_t e = s_e;
    const uint64_t tag = (e & 0xffffffffull) << 32;   // e >= 1: never the zeroed window's tag
    const size_t row = (size_t)n * 8, half = row * c.world;
    const size_t par = stage_off + (e & 1) * half;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint64_t w = tag | to_bits<T>(__ldcg(buf + i));
        const size_t at = par + (size_t)c.rank * row + (size_t)i * 8;
        for_each_rank(c, [at, w](int, char *b) { st_relaxed_sys((uint64_t *)(b + at), w); });
    }
    const uint64_t *rows = (const uint64_t *)(c.self + par);
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        T acc{};
        for (int q = 0; q < c.world; ++q) {
            // the word is the data: no acquire fence needed
            const uint64_t w = spin_until<false>(rows + (size_t)q * n + i,
                                                 [tag](uint64_t v) { return (v & 0xffffffff00000000ull) == tag; });
            const T v = from_bits<T>((uint32_t)w);
            acc = q == 0 ? v : acc + v;
        }
        buf[i] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) *count(c, slot) = e;
}

}  // namespace peer
}  // namespace jacc_k
