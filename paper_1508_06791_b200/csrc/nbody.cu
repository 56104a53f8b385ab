// nbody.cu -- one symplectic-Euler step of softened direct-sum gravity
// (north_star; not in PAPER.md -- SURVEY D1, reading R16):
//   a_i = G sum_j m_j (x_j - x_i) / (|x_j - x_i|^2 + eps2)^{3/2}
//   v_i <- v_i + a_i dt;   x_i <- x_i + v_i dt
// pos_src holds all n_src bodies (x, y, z, m); targets are bodies
// tgt_offset .. tgt_offset + n_tgt - 1 (a rank's shard in SPMD, R17).
//
// sm_100a design (FP32-pipe bound: 11-12 fp32 ops + 1 MUFU.RSQ per interaction):
//   * work unit = (64 threads x 2P targets) x (one chunk of kChunk = 2048
//     sources).  The chunk size is a constant, so every rank of a sharded run
//     sums a target's sources in exactly the same groups as one GPU does
//     (bitwise shard invariance, §8(e)); it is small so that even a 1/8
//     shard has several waves of units (2^17 bodies: 21.9k units = 24.6 waves
//     of 888 resident blocks; measured 6.54 ms vs 6.71 ms with 8192-source
//     chunks = 6.2 waves).  Targets per thread (P pairs) only decide which
//     thread computes a target, never the order of its sum, so P is chosen
//     per launch from the wave count (P = 3 full size, P = 2 for shards);
//   * sources stream through shared memory in tiles of 256, stored
//     duplicated as (x,x,y,y),(z,z,m,m) so one LDS.128 yields the operand
//     pairs of the paired FP32 instructions; grids only a few waves deep
//     (target shards) use a double-buffered kernel, the next tile arriving
//     by cp.async while the current one is summed;
//   * each thread holds P target PAIRS in registers and uses the sm_100
//     FADD2/FFMA2/FMUL2 (FMA-heavy pipe): 12 paired ops (11 on equal-mass
//     tiles) + 2 MUFU.RSQ per pair and source, half the FP32 issue slots of
//     scalar code;
//     measured alternatives (scalar FP32 on the other pipe for some targets,
//     an lg2/ex2 path that moves work to the MUFU) were slower;
//   * accumulation is TILE-PARTIAL (each tile summed separately, then added
//     in tile order), chunk partials go to a workspace and a second kernel
//     adds the chunks in order and applies kick + drift;
//   * the self term is included: x_j - x_i = 0 with eps2 > 0 contributes 0;
//     padding sources (j >= n_src) have m = 0 at the origin (contribute 0).
//   * JACC_GRAPH_P2P fusion (reading R23): when the graph's next task
//     all-gathers pos_out, the finish kernel performs it -- every thread
//     stores its target's new position into its own slot of every rank's
//     gathered buffer over NVLink as soon as it is computed, and the last
//     block waits until every rank's positions have arrived.  The all-gather
//     costs no separate launch and its transfer overlaps the kick/drift.
#include "common.cuh"
#include "kernels.h"
#include "peer.cuh"

namespace jacc_k {
namespace {

constexpr int kBlock = 64;
constexpr int kTile = 256;                    // sources per shared-memory tile
constexpr int kChunk = 2048;                  // sources per work unit (fixed: shard invariance)

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// Sum of one shared-memory tile of sources into the tile partials t* of the
// thread's P target pairs, with the paired FP32 instructions (FADD2/FFMA2/
// FMUL2, FMA-heavy pipe): per pair and source 3 FADD2 + 3 FFMA2 (r^2) +
// 2 MUFU.RSQ + 3 FMUL2 (s = m inv^3) + 3 FFMA2 (t += d s).  kEqualMass: every
// source of the tile has the same mass m, so m is factored out of the tile
// sum -- s = inv^3 takes 2 FMUL2 (11 instead of 12 FP32 lane-ops per
// interaction) and the caller scales the tile partial by m once.
template <int P, int UNR, bool kEqualMass>
__device__ __forceinline__ void tile_sum(const float4 *tile, const float2 (&nx)[P], const float2 (&ny)[P],
                                         const float2 (&nz)[P], float2 e2, float2 (&tx)[P], float2 (&ty)[P],
                                         float2 (&tz)[P]) {
#pragma unroll UNR
    for (int s = 0; s < kTile; ++s) {
        const float4 A = tile[2 * s], B = tile[2 * s + 1];
        const float2 xj = f2(A.x, A.y), yj = f2(A.z, A.w), zj = f2(B.x, B.y), mj = f2(B.z, B.w);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const float2 dx = __fadd2_rn(xj, nx[p]), dy = __fadd2_rn(yj, ny[p]), dz = __fadd2_rn(zj, nz[p]);
            float2 r2 = __ffma2_rn(dx, dx, e2);
            r2 = __ffma2_rn(dy, dy, r2);
            r2 = __ffma2_rn(dz, dz, r2);
            const float2 inv = f2(rsqrt_approx(r2.x), rsqrt_approx(r2.y));
            const float2 sc = kEqualMass ? __fmul2_rn(__fmul2_rn(inv, inv), inv)
                                         : __fmul2_rn(__fmul2_rn(mj, inv), __fmul2_rn(inv, inv));
            tx[p] = __ffma2_rn(dx, sc, tx[p]);
            ty[p] = __ffma2_rn(dy, sc, ty[p]);
            tz[p] = __ffma2_rn(dz, sc, tz[p]);
        }
    }
}

// One work unit: kBlock * 2P targets x one chunk of sources.  Every thread
// holds P target PAIRS (paired FP32 instructions: half the issue slots of
// scalar code for the same arithmetic).  Target k of thread tid is
// t0 + tid + k * kBlock.  Sources stream through shared memory one tile at a
// time; a tile whose sources all have the same mass takes the equal-mass sum
// (for a power-of-two mass, e.g. the workload's m = 1/N, its result is
// bitwise identical to the general sum: scaling by 2^k commutes with every
// rounding), any other tile (mixed masses, zero-mass padding) the general one.
template <int P, int MINB, int UNR>
__global__ void __launch_bounds__(kBlock, MINB) nbody_partial_kernel(const float4 *__restrict__ pos_src, int64_t n_src,
                                                               int64_t n_tgt, int64_t tgt_offset, float eps2,
                                                               float4 *__restrict__ part) {
    constexpr int T = 2 * P;
    __shared__ float4 tile[2 * kTile];    // per source: (x, x, y, y), (z, z, m, m)
    const int64_t t0 = (int64_t)blockIdx.x * (kBlock * T);
    const int64_t j_begin = (int64_t)blockIdx.y * kChunk;
    const int64_t j_end = min(j_begin + kChunk, n_src);
    float2 nx[P], ny[P], nz[P], ax[P], ay[P], az[P];    // nx = -x of the target pair
    auto load_t = [&](int k) {
        const int64_t t = t0 + threadIdx.x + k * kBlock;
        return t < n_tgt ? pos_src[tgt_offset + t] : make_float4(0.f, 0.f, 0.f, 0.f);
    };
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const float4 a = load_t(2 * p), b = load_t(2 * p + 1);
        nx[p] = f2(-a.x, -b.x); ny[p] = f2(-a.y, -b.y); nz[p] = f2(-a.z, -b.z);
        ax[p] = ay[p] = az[p] = f2(0.f, 0.f);
    }
    const float2 e2 = f2(eps2, eps2);
    for (int64_t j0 = j_begin; j0 < j_end; j0 += kTile) {
        const float m0 = pos_src[j0].w;
        bool same = true;
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kTile / kBlock; ++q) {
            const int s = threadIdx.x + q * kBlock;
            const int64_t j = j0 + s;
            const float4 v = j < j_end ? pos_src[j] : make_float4(0.f, 0.f, 0.f, 0.f);
            same &= v.w == m0;
            tile[2 * s] = make_float4(v.x, v.x, v.y, v.y);
            tile[2 * s + 1] = make_float4(v.z, v.z, v.w, v.w);
        }
        const bool equal_mass = __syncthreads_and(same);
        float2 tx[P], ty[P], tz[P];
#pragma unroll
        for (int p = 0; p < P; ++p) tx[p] = ty[p] = tz[p] = f2(0.f, 0.f);
        if (equal_mass) {
            tile_sum<P, UNR, true>(tile, nx, ny, nz, e2, tx, ty, tz);
            const float2 m2 = f2(m0, m0);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                ax[p] = __ffma2_rn(tx[p], m2, ax[p]);
                ay[p] = __ffma2_rn(ty[p], m2, ay[p]);
                az[p] = __ffma2_rn(tz[p], m2, az[p]);
            }
        } else {
            tile_sum<P, UNR, false>(tile, nx, ny, nz, e2, tx, ty, tz);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                ax[p] = __fadd2_rn(ax[p], tx[p]);
                ay[p] = __fadd2_rn(ay[p], ty[p]);
                az[p] = __fadd2_rn(az[p], tz[p]);
            }
        }
    }
    float4 *out = part + (int64_t)blockIdx.y * n_tgt;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int64_t ta = t0 + threadIdx.x + (2 * p) * kBlock, tb = ta + kBlock;
        if (ta < n_tgt) out[ta] = make_float4(ax[p].x, ay[p].x, az[p].x, 0.f);
        if (tb < n_tgt) out[tb] = make_float4(ax[p].y, ay[p].y, az[p].y, 0.f);
    }
}

// One work unit of the double-buffered kernel: kBlock * 2P targets starting at
// t0, sources of chunk `chunk`; tile / stage are the block's shared buffers.
template <int P, int UNR>
__device__ __forceinline__ void partial_unit_db(const float4 *__restrict__ pos_src, int64_t n_src, int64_t n_tgt,
                                                int64_t tgt_offset, float eps2, float4 *__restrict__ part, int64_t t0,
                                                int64_t chunk, float4 (*tile)[2 * kTile], float4 *stage) {
    const int64_t j_begin = chunk * kChunk;
    const int64_t j_end = min(j_begin + kChunk, n_src);
    float2 nx[P], ny[P], nz[P], ax[P], ay[P], az[P];    // nx = -x of the target pair
    auto load_t = [&](int k) {
        const int64_t t = t0 + threadIdx.x + k * kBlock;
        return t < n_tgt ? pos_src[tgt_offset + t] : make_float4(0.f, 0.f, 0.f, 0.f);
    };
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const float4 a = load_t(2 * p), b = load_t(2 * p + 1);
        nx[p] = f2(-a.x, -b.x); ny[p] = f2(-a.y, -b.y); nz[p] = f2(-a.z, -b.z);
        ax[p] = ay[p] = az[p] = f2(0.f, 0.f);
    }
    const float2 e2 = f2(eps2, eps2);
    // a thread stages and expands the same sources s = tid + q * kBlock, so it
    // only waits for its own copies; padding (j >= j_end) is zero-filled
    auto fetch = [&](int64_t j0) {
#pragma unroll
        for (int q = 0; q < kTile / kBlock; ++q) {
            const int s = threadIdx.x + q * kBlock;
            const int64_t j = j0 + s;
            const unsigned dst = (unsigned)__cvta_generic_to_shared(&stage[s]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(pos_src + (j < j_end ? j : j0)),
                         "r"(j < j_end ? 16 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto expand = [&](int b, float m0) {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        bool same = true;
#pragma unroll
        for (int q = 0; q < kTile / kBlock; ++q) {
            const int s = threadIdx.x + q * kBlock;
            const float4 v = stage[s];
            same &= v.w == m0;
            tile[b][2 * s] = make_float4(v.x, v.x, v.y, v.y);
            tile[b][2 * s + 1] = make_float4(v.z, v.z, v.w, v.w);
        }
        return same;
    };
    __syncthreads();   // the previous unit of this block is done with tile / stage
    fetch(j_begin);
    float m0 = pos_src[j_begin].w;
    bool equal_mass = __syncthreads_and(expand(0, m0));
    int buf = 0;
    for (int64_t j0 = j_begin; j0 < j_end; j0 += kTile) {
        const int64_t jn = j0 + kTile;
        const bool more = jn < j_end;   // block-uniform
        float m0n = 0.f;
        if (more) {
            fetch(jn);
            m0n = pos_src[jn].w;
        }
        float2 tx[P], ty[P], tz[P];
#pragma unroll
        for (int p = 0; p < P; ++p) tx[p] = ty[p] = tz[p] = f2(0.f, 0.f);
        if (equal_mass) {
            tile_sum<P, UNR, true>(tile[buf], nx, ny, nz, e2, tx, ty, tz);
            const float2 m2 = f2(m0, m0);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                ax[p] = __ffma2_rn(tx[p], m2, ax[p]);
                ay[p] = __ffma2_rn(ty[p], m2, ay[p]);
                az[p] = __ffma2_rn(tz[p], m2, az[p]);
            }
        } else {
            tile_sum<P, UNR, false>(tile[buf], nx, ny, nz, e2, tx, ty, tz);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                ax[p] = __fadd2_rn(ax[p], tx[p]);
                ay[p] = __fadd2_rn(ay[p], ty[p]);
                az[p] = __fadd2_rn(az[p], tz[p]);
            }
        }
        if (!more) break;
        equal_mass = __syncthreads_and(expand(buf ^ 1, m0n));
        m0 = m0n;
        buf ^= 1;
    }
    float4 *out = part + chunk * n_tgt;
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const int64_t ta = t0 + threadIdx.x + (2 * p) * kBlock, tb = ta + kBlock;
        if (ta < n_tgt) out[ta] = make_float4(ax[p].x, ay[p].x, az[p].x, 0.f);
        if (tb < n_tgt) out[tb] = make_float4(ax[p].y, ay[p].y, az[p].y, 0.f);
    }
}

// Double-buffered variant of the kernel above: two tile buffers, the next
// tile's raw float4s arriving by cp.async into `stage` while the current tile
// is summed, one barrier per tile.  Measured (ms per step at 2^17 bodies,
// target shards 1/2/4/8): single 6.103 / 3.382 / 1.724 / 0.836, double
// 6.201 / 3.104 / 1.651 / 0.846 -- double buffering pays when the grid is
// only a few waves deep (SMs then hold few blocks and a tile load's L2
// latency is not covered by the others); its per-tile overhead costs 1.5 %
// when many waves keep every SM full.  (Kept as a separate kernel: a merged
// template with both loops compiled 2 % slower in both modes.)
template <int P, int MINB, int UNR>
__global__ void __launch_bounds__(kBlock, MINB) nbody_partial_db_kernel(const float4 *__restrict__ pos_src, int64_t n_src,
                                                               int64_t n_tgt, int64_t tgt_offset, float eps2,
                                                               float4 *__restrict__ part) {
    __shared__ float4 tile[2][2 * kTile];
    __shared__ float4 stage[kTile];
    partial_unit_db<P, UNR>(pos_src, n_src, n_tgt, tgt_offset, eps2, part, (int64_t)blockIdx.x * (kBlock * 2 * P),
                            blockIdx.y, tile, stage);
}

// Mixed grid for target shards a few waves deep: the first n_big units (in
// dispatch order) cover targets [0, t_big) with 3 target pairs per thread --
// the most efficient per interaction -- and fill whole waves; the remaining
// targets follow as 1-pair units, a third of the size, so the last, partial
// wave is made of small units instead of leaving most SMs idle behind a few
// large ones.  1-D grid; unit u < n_big: target block u % nb_big of chunk
// u / nb_big.  Which thread computes a target never changes the order of its
// sum (chunk partials, tile order), so results are bitwise those of any
// other variant.
template <int MINB, int UNR>
__global__ void __launch_bounds__(kBlock, MINB) nbody_partial_mixed_kernel(const float4 *__restrict__ pos_src,
                                                                  int64_t n_src, int64_t n_tgt, int64_t tgt_offset,
                                                                  float eps2, float4 *__restrict__ part, int nb_big,
                                                                  int64_t n_big, int64_t t_big, int nb_small) {
    __shared__ float4 tile[2][2 * kTile];
    __shared__ float4 stage[kTile];
    const int64_t u = blockIdx.x;
    if (u < n_big) {
        partial_unit_db<3, UNR>(pos_src, n_src, n_tgt, tgt_offset, eps2, part, (u % nb_big) * (kBlock * 6),
                                u / nb_big, tile, stage);
    } else {
        const int64_t v = u - n_big;
        partial_unit_db<1, UNR>(pos_src, n_src, n_tgt, tgt_offset, eps2, part, t_big + (v % nb_small) * (kBlock * 2),
                                v / nb_small, tile, stage);
    }
}

// ---- chunk sum (in chunk order) + kick + drift ---------------------------
// kPeer: also the all-gather of pos_out into offset pop.off of every rank's
// window (rank r's targets at [r n_tgt, (r+1) n_tgt)).  Receivers publish
// "ready" first: this kernel runs after the step's partial kernel, the last
// reader of the gathered buffer, and only reads its own slot of it.
// Four lanes per target: lane q adds the chunk partials of its quarter of
// the chunks in chunk order, then lane 0 of the quad combines the quarters in
// a fixed order, ((q0 + q1) + q2) + q3 -- the same function of the partials
// for every shard size (bitwise shard invariance) with 4x the threads and
// loads in flight of one lane per target (a 1/8 shard has only 2^14
// targets: one lane each left the kernel latency-bound).
constexpr int kFinishLanes = 4;

template <bool kPeer>
__global__ void __launch_bounds__(256) nbody_finish_kernel(const float4 *__restrict__ part, int nchunks,
                                                           const float4 *__restrict__ pos_src, int64_t tgt_offset,
                                                           float4 *__restrict__ vel, float4 *__restrict__ pos_out,
                                                           int64_t n_tgt, float dt, float G, PeerOp pop) {
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t t = gt / kFinishLanes;
    const int q = (int)(gt % kFinishLanes);
    uint64_t e = 0;
    if (kPeer) {
        e = peer::epoch(pop.ctx, pop.slot);
        if (blockIdx.x == 0 && threadIdx.x == 0) peer::signal_all(pop.ctx, peer::kReadyOff, pop.slot, e);
    }
    float3 s3 = make_float3(0.f, 0.f, 0.f);
    if (t < n_tgt) {
        const int per = (nchunks + kFinishLanes - 1) / kFinishLanes;
        const int c0 = q * per, c1 = min(nchunks, c0 + per);
        const float4 *pt = part + t;
        int c = c0;
        for (; c + 8 <= c1; c += 8) {   // 8 independent loads in flight, added in chunk order
            float4 b[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) b[k] = __ldg(pt + (int64_t)(c + k) * n_tgt);
#pragma unroll
            for (int k = 0; k < 8; ++k) { s3.x += b[k].x; s3.y += b[k].y; s3.z += b[k].z; }
        }
        for (; c < c1; ++c) {
            const float4 b = __ldg(pt + (int64_t)c * n_tgt);
            s3.x += b.x; s3.y += b.y; s3.z += b.z;
        }
    }
    // quad combine in lane order (all lanes of the warp take part)
    const unsigned lane = threadIdx.x & 31, base = lane & ~(unsigned)(kFinishLanes - 1);
    float3 a = s3;
#pragma unroll
    for (int k = 1; k < kFinishLanes; ++k) {
        a.x += __shfl_sync(0xffffffffu, s3.x, base + k);
        a.y += __shfl_sync(0xffffffffu, s3.y, base + k);
        a.z += __shfl_sync(0xffffffffu, s3.z, base + k);
    }
    float4 np = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool owner = t < n_tgt && q == 0;
    if (owner) {
        float4 v = vel[t];
        v.x = fmaf(G * a.x, dt, v.x);
        v.y = fmaf(G * a.y, dt, v.y);
        v.z = fmaf(G * a.z, dt, v.z);
        vel[t] = v;
        const float4 p = pos_src[tgt_offset + t];
        np = make_float4(fmaf(v.x, dt, p.x), fmaf(v.y, dt, p.y), fmaf(v.z, dt, p.z), p.w);
        pos_out[t] = np;
    }
    if (!kPeer) return;
    const PeerCtx &c = pop.ctx;
    const size_t slot_off = (size_t)pop.off + ((size_t)c.rank * n_tgt + t) * sizeof(float4);
    peer::for_each_rank(c, [&](int r, char *b) {
        if (r != c.rank) peer::block_wait(c, peer::kReadyOff, pop.slot, r, e);
        if (owner) *(float4 *)(b + slot_off) = np;
    });
    if (!peer::grid_last(c, pop.slot)) return;
    if (threadIdx.x == 0) peer::publish_data(c, pop.slot, e);
    peer::wait_all_data(c, pop.slot, e);
}

typedef void (*partial_fn)(const float4 *, int64_t, int64_t, int64_t, float, float4 *);
struct Variant { partial_fn fn; int tpt; };

// Source loop unrolled by 4 (re-measured with the equal-mass path, ms per
// 2^17 step: P3/unroll 4 6.087, unroll 1 6.52, 2 6.20, 8 6.19; P4/2 6.43;
// P2/8 6.34).  P = 3 pairs (152
// registers, 6 blocks/SM) is the fastest per interaction at 2^17 bodies
// (6.54 ms vs 6.67 for P = 2 at 10 blocks/SM, 7.0 for P = 4); P = 2 and
// P = 1 give more, smaller units when a shard has few targets.  The variant
// with the fewest waves x resident targets per SM wins (ties: larger P);
// grids under 16 waves (of the P = 3 single-buffered kernel) choose among
// the double-buffered kernels.
Variant variant(int64_t n_tgt, int64_t nchunks) {
    const Variant single[3] = {{nbody_partial_kernel<3, 1, 4>, 6}, {nbody_partial_kernel<2, 10, 4>, 4},
                               {nbody_partial_kernel<1, 16, 4>, 2}};
    const Variant dbl[3] = {{nbody_partial_db_kernel<3, 1, 4>, 6}, {nbody_partial_db_kernel<2, 10, 4>, 4},
                            {nbody_partial_db_kernel<1, 16, 4>, 2}};
    const int sms = sm_count();
    // waves of a family's variant i, and its cost = waves (rounded up) x
    // resident targets per SM (the time of one wave is ~ proportional to it)
    auto waves = [&](const Variant *fam, int i, double *cost) -> double {
        const int occ = blocks_per_sm((const void *)fam[i].fn, kBlock, 0);
        const int64_t per_block = (int64_t)kBlock * fam[i].tpt;
        const int64_t units = (n_tgt + per_block - 1) / per_block * nchunks;
        const int64_t slots = (int64_t)occ * sms;
        *cost = (double)((units + slots - 1) / slots) * occ * per_block;
        return (double)units / slots;
    };
    double c;
    const bool deep = waves(single, 0, &c) >= 16.0;   // many waves: every SM stays full
    const Variant *fam = deep ? single : dbl;
    int best = 0;
    double best_cost = 0;
    for (int i = 0; i < 3; ++i) {
        if ((n_tgt + (int64_t)kBlock * fam[i].tpt - 1) / ((int64_t)kBlock * fam[i].tpt) > 0x7fffffff) continue;
        waves(fam, i, &c);
        if (best_cost == 0 || c < best_cost * 0.97) { best = i; best_cost = c; }
    }
    return fam[best];
}

// Mixed grid (nbody_partial_mixed_kernel) for grids a few waves deep: whole
// waves of 3-pair units, the rest of the targets as 1-pair units.
struct Mixed {
    int nb_big, nb_small;
    int64_t n_big, t_big;
};
bool mixed_plan(int64_t n_tgt, int64_t nchunks, Mixed *m) {
    const int sms = sm_count();
    const int occ = blocks_per_sm((const void *)nbody_partial_mixed_kernel<1, 4>, kBlock, 0);
    const int64_t slots = (int64_t)occ * sms;
    const int64_t big = kBlock * 6, small = kBlock * 2;
    const int64_t big_units = (n_tgt + big - 1) / big * nchunks;
    const int64_t full_waves = big_units / slots;
    // up to 8 waves of 3-pair units; deeper grids already keep the SMs full
    // (measured, ms per step at 2^17 bodies, target shard 1/2 / 1/4 / 1/8:
    // single-variant kernels 3.054 / 1.663 / 0.848, mixed 3.118 / 1.589 / 0.817)
    if (full_waves < 1 || big_units > 8 * slots) return false;
    int64_t nb_big = full_waves * slots / nchunks;
    if (nb_big * big > n_tgt) nb_big = n_tgt / big;
    if (nb_big < 1) return false;
    m->nb_big = (int)nb_big;
    m->n_big = nb_big * nchunks;
    m->t_big = nb_big * big;
    m->nb_small = (int)((n_tgt - m->t_big + small - 1) / small);
    return m->n_big + (int64_t)m->nb_small * nchunks < 0x7fffffff;
}

}  // namespace

size_t nbody_ws_bytes(int64_t n_src, int64_t n_tgt) {
    const int64_t nchunks = (n_src + kChunk - 1) / kChunk;
    return (size_t)(nchunks > 0 ? nchunks : 1) * (size_t)(n_tgt > 0 ? n_tgt : 1) * sizeof(float4);
}

cudaError_t nbody_step_f32(const float4 *pos_src, int64_t n_src, float4 *vel, float4 *pos_out, int64_t n_tgt,
                           const jacc_nbody_params_t *p, void *ws, const jacc_schedule_t *, cudaStream_t st,
                           int *launches, const PeerOp *pop) {
    if (pop && n_tgt <= 0) return cudaErrorInvalidValue;   // the runtime only fuses n_tgt > 0
    if (n_tgt <= 0) return cudaSuccess;
    float4 *part = (float4 *)ws;
    const int64_t nchunks = (n_src + kChunk - 1) / kChunk;
    if (nchunks == 0) {   // no sources: a = 0
        cudaError_t e = cudaMemsetAsync(part, 0, n_tgt * sizeof(float4), st);
        if (e != cudaSuccess) return e;
    } else {
        if (nchunks > 65535) return cudaErrorInvalidConfiguration;   // > 134M sources: shard further
        Mixed mx;
        if (mixed_plan(n_tgt, nchunks, &mx)) {
            nbody_partial_mixed_kernel<1, 4><<<(unsigned)(mx.n_big + (int64_t)mx.nb_small * nchunks), kBlock, 0, st>>>(
                pos_src, n_src, n_tgt, p->tgt_offset, p->eps2, part, mx.nb_big, mx.n_big, mx.t_big, mx.nb_small);
        } else {
            const Variant v = variant(n_tgt, nchunks);
            const int64_t per_block = (int64_t)kBlock * v.tpt;
            dim3 grid((unsigned)((n_tgt + per_block - 1) / per_block), (unsigned)nchunks);
            v.fn<<<grid, kBlock, 0, st>>>(pos_src, n_src, n_tgt, p->tgt_offset, p->eps2, part);
        }
        ++*launches;
    }
    auto fin = pop ? nbody_finish_kernel<true> : nbody_finish_kernel<false>;
    fin<<<(unsigned)((n_tgt * kFinishLanes + 255) / 256), 256, 0, st>>>(part, nchunks > 0 ? (int)nchunks : 1, pos_src,
                                                         p->tgt_offset, vel, pos_out, n_tgt, p->dt, p->G,
                                                         pop ? *pop : PeerOp{});
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
