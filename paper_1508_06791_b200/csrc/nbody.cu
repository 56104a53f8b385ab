// nbody.cu -- one symplectic-Euler step of softened direct-sum gravity
// (north_star; not in PAPER.md -- SURVEY D1, reading R16):
//   a_i = G sum_j m_j (x_j - x_i) / (|x_j - x_i|^2 + eps2)^{3/2}
//   v_i <- v_i + a_i dt;   x_i <- x_i + v_i dt
// pos_src holds all n_src bodies (x, y, z, m); targets are bodies
// tgt_offset .. tgt_offset + n_tgt - 1 (a rank's shard in SPMD, R17).
//
// sm_100a design (FP32-pipe bound: 12 fp32 ops + 1 MUFU.RSQ per interaction):
//   * work unit = (64 threads x 6 targets) x (one chunk of kChunk = 8192
//     sources); the chunk size depends on nothing but the source count, so
//     every rank of a sharded run sums a target's sources in exactly the same
//     groups as one GPU does (bitwise shard invariance, §8(e)), and 2^17
//     bodies give ~5.5k units -- 37 per SM, the 148 SMs finish together;
//   * sources stream through shared memory in tiles of 256, stored
//     duplicated as (x,x,y,y),(z,z,m,m) so one LDS.128 yields the operand
//     pairs of the paired FP32 instructions;
//   * each thread holds 3 target PAIRS in registers and uses the sm_100
//     FADD2/FFMA2/FMUL2 (FMA-heavy pipe): 12 paired ops + 2 MUFU.RSQ per
//     pair and source, half the FP32 issue slots of scalar code;
//     measured alternatives (scalar FP32 on the other pipe for some targets,
//     an lg2/ex2 path that moves work to the MUFU) were slower;
//   * accumulation is TILE-PARTIAL (each tile summed separately, then added
//     in tile order), chunk partials go to a workspace and a second kernel
//     adds the chunks in order and applies kick + drift;
//   * the self term is included: x_j - x_i = 0 with eps2 > 0 contributes 0;
//     padding sources (j >= n_src) have m = 0 at the origin (contribute 0).
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {

constexpr int kBlock = 64;
constexpr int kTile = 256;                    // sources per shared-memory tile
constexpr int kChunk = 8192;                  // sources per work unit

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// One work unit: kBlock * 2P targets x one chunk of sources.  Every thread
// holds P target PAIRS and uses the paired FP32 instructions
// (FADD2/FFMA2/FMUL2, FMA-heavy pipe) -- half the FP32 issue slots of scalar
// code for the same arithmetic: per pair and source 12 paired ops + 2
// MUFU.RSQ.  Target k of thread tid is t0 + tid + k * kBlock.
template <int P, int MINB, int UNR>
__global__ void __launch_bounds__(kBlock, MINB) nbody_partial_kernel(const float4 *__restrict__ pos_src, int64_t n_src,
                                                               int64_t n_tgt, int64_t tgt_offset, float eps2,
                                                               float4 *__restrict__ part) {
    constexpr int T = 2 * P;
    constexpr int TW = 2;                 // float4 words per source in the tile
    __shared__ float4 tile[TW * kTile];   // (x, x, y, y), (z, z, m, m)
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
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kTile / kBlock; ++q) {
            const int s = threadIdx.x + q * kBlock;
            const int64_t j = j0 + s;
            const float4 v = j < j_end ? pos_src[j] : make_float4(0.f, 0.f, 0.f, 0.f);
            tile[TW * s] = make_float4(v.x, v.x, v.y, v.y);
            tile[TW * s + 1] = make_float4(v.z, v.z, v.w, v.w);
        }
        __syncthreads();
        float2 tx[P], ty[P], tz[P];
#pragma unroll
        for (int p = 0; p < P; ++p) tx[p] = ty[p] = tz[p] = f2(0.f, 0.f);
#pragma unroll UNR
        for (int s = 0; s < kTile; ++s) {
            const float4 A = tile[TW * s], B = tile[TW * s + 1];
            const float2 xj = f2(A.x, A.y), yj = f2(A.z, A.w), zj = f2(B.x, B.y), mj = f2(B.z, B.w);
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const float2 dx = __fadd2_rn(xj, nx[p]), dy = __fadd2_rn(yj, ny[p]), dz = __fadd2_rn(zj, nz[p]);
                float2 r2 = __ffma2_rn(dx, dx, e2);
                r2 = __ffma2_rn(dy, dy, r2);
                r2 = __ffma2_rn(dz, dz, r2);
                const float2 inv = f2(rsqrt_approx(r2.x), rsqrt_approx(r2.y));
                const float2 sc = __fmul2_rn(__fmul2_rn(mj, inv), __fmul2_rn(inv, inv));
                tx[p] = __ffma2_rn(dx, sc, tx[p]);
                ty[p] = __ffma2_rn(dy, sc, ty[p]);
                tz[p] = __ffma2_rn(dz, sc, tz[p]);
            }
        }
#pragma unroll
        for (int p = 0; p < P; ++p) {
            ax[p] = __fadd2_rn(ax[p], tx[p]);
            ay[p] = __fadd2_rn(ay[p], ty[p]);
            az[p] = __fadd2_rn(az[p], tz[p]);
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

// ---- chunk sum (in chunk order) + kick + drift ---------------------------
__global__ void __launch_bounds__(256) nbody_finish_kernel(const float4 *__restrict__ part, int nchunks,
                                                           const float4 *__restrict__ pos_src, int64_t tgt_offset,
                                                           float4 *__restrict__ vel, float4 *__restrict__ pos_out,
                                                           int64_t n_tgt, float dt, float G) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tgt) return;
    float4 a = part[t];
    for (int c = 1; c < nchunks; ++c) {
        const float4 b = part[(int64_t)c * n_tgt + t];
        a.x += b.x; a.y += b.y; a.z += b.z;
    }
    float4 v = vel[t];
    v.x = fmaf(G * a.x, dt, v.x);
    v.y = fmaf(G * a.y, dt, v.y);
    v.z = fmaf(G * a.z, dt, v.z);
    vel[t] = v;
    const float4 p = pos_src[tgt_offset + t];
    pos_out[t] = make_float4(fmaf(v.x, dt, p.x), fmaf(v.y, dt, p.y), fmaf(v.z, dt, p.z), p.w);
}

typedef void (*partial_fn)(const float4 *, int64_t, int64_t, int64_t, float, float4 *);
struct Variant { partial_fn fn; int tpt; };

// 3 target pairs per thread, source loop unrolled by 4: measured best on B200
// at 2^17 bodies (ms/step: P=3 6.70, P=2 6.75, P=4 7.01; unroll 2/8 slower).
Variant variant() { return Variant{nbody_partial_kernel<3, 1, 4>, 6}; }

}  // namespace

size_t nbody_ws_bytes(int64_t n_src, int64_t n_tgt) {
    const int64_t nchunks = (n_src + kChunk - 1) / kChunk;
    return (size_t)(nchunks > 0 ? nchunks : 1) * (size_t)(n_tgt > 0 ? n_tgt : 1) * sizeof(float4);
}

cudaError_t nbody_step_f32(const float4 *pos_src, int64_t n_src, float4 *vel, float4 *pos_out, int64_t n_tgt,
                           const jacc_nbody_params_t *p, void *ws, const jacc_schedule_t *, cudaStream_t st,
                           int *launches) {
    if (n_tgt <= 0) return cudaSuccess;
    float4 *part = (float4 *)ws;
    const int64_t nchunks = (n_src + kChunk - 1) / kChunk;
    if (nchunks == 0) {   // no sources: a = 0
        cudaError_t e = cudaMemsetAsync(part, 0, n_tgt * sizeof(float4), st);
        if (e != cudaSuccess) return e;
    } else {
        const Variant v = variant();
        const int64_t per_block = (int64_t)kBlock * v.tpt;
        dim3 grid((unsigned)((n_tgt + per_block - 1) / per_block), (unsigned)nchunks);
        v.fn<<<grid, kBlock, 0, st>>>(pos_src, n_src, n_tgt, p->tgt_offset, p->eps2, part);
        ++*launches;
    }
    nbody_finish_kernel<<<(unsigned)((n_tgt + 255) / 256), 256, 0, st>>>(part, nchunks > 0 ? (int)nchunks : 1,
                                                                         pos_src, p->tgt_offset, vel, pos_out, n_tgt,
                                                                         p->dt, p->G);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
