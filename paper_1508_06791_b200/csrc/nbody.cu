// nbody.cu -- one symplectic-Euler step of softened direct-sum gravity
// (north_star; not in PAPER.md -- SURVEY D1, reading R16):
//   a_i = G sum_j m_j (x_j - x_i) / (|x_j - x_i|^2 + eps2)^{3/2}
//   v_i <- v_i + a_i dt;   x_i <- x_i + v_i dt
// pos_src holds all n_src bodies (x, y, z, m); targets are bodies
// tgt_offset .. tgt_offset + n_tgt - 1 (a rank's shard in SPMD, R17).
//
// sm_100a design (FP32-pipe bound, 12 fp32 ops + 1 MUFU.RSQ / interaction):
//   * sources stream through shared memory in tiles of kTile bodies (float4),
//     every thread keeps kTpt targets in registers, so each LDS.128 of a
//     source feeds kTpt interactions;
//   * accumulation is TILE-PARTIAL: each tile's contributions are summed
//     separately, then added to the running total in tile order (the
//     accuracy of a blocked sum, SURVEY §8(c)-N [exp]);
//   * the self term is included: x_j - x_i = 0 and eps2 > 0 make it exactly 0;
//   * padding sources beyond n_src have m = 0 at the origin (contribute 0).
// The j order is the global order for every target, so a rank computing a
// shard gets the same bits as one GPU computing everything (§8(e)).
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {

constexpr int kBlock = 128;
constexpr int kTpt = 2;                 // targets per thread
constexpr int kTile = kBlock;           // sources per shared-memory tile

__device__ __forceinline__ float rsqrt_approx(float x) {
    float y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __launch_bounds__(kBlock) nbody_kernel(const float4 *__restrict__ pos_src, int64_t n_src,
                                                       float4 *__restrict__ vel, float4 *__restrict__ pos_out,
                                                       int64_t n_tgt, int64_t tgt_offset, float dt, float eps2,
                                                       float G) {
    __shared__ float4 tile[kTile];
    const int64_t base = (int64_t)blockIdx.x * (kBlock * kTpt);
    float xi[kTpt], yi[kTpt], zi[kTpt];
    float ax[kTpt], ay[kTpt], az[kTpt];
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
        const int64_t t = base + threadIdx.x + k * kBlock;
        float4 p = make_float4(0.f, 0.f, 0.f, 0.f);
        if (t < n_tgt) p = pos_src[tgt_offset + t];
        xi[k] = p.x; yi[k] = p.y; zi[k] = p.z;
        ax[k] = ay[k] = az[k] = 0.f;
    }
    for (int64_t j0 = 0; j0 < n_src; j0 += kTile) {
        const int64_t j = j0 + threadIdx.x;
        tile[threadIdx.x] = j < n_src ? pos_src[j] : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        float tx[kTpt], ty[kTpt], tz[kTpt];
#pragma unroll
        for (int k = 0; k < kTpt; ++k) tx[k] = ty[k] = tz[k] = 0.f;
#pragma unroll 8
        for (int s = 0; s < kTile; ++s) {
            const float4 q = tile[s];
#pragma unroll
            for (int k = 0; k < kTpt; ++k) {
                const float dx = q.x - xi[k], dy = q.y - yi[k], dz = q.z - zi[k];
                const float r2 = fmaf(dz, dz, fmaf(dy, dy, fmaf(dx, dx, eps2)));
                const float inv = rsqrt_approx(r2);
                const float sc = q.w * inv * inv * inv;
                tx[k] = fmaf(dx, sc, tx[k]);
                ty[k] = fmaf(dy, sc, ty[k]);
                tz[k] = fmaf(dz, sc, tz[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < kTpt; ++k) { ax[k] += tx[k]; ay[k] += ty[k]; az[k] += tz[k]; }
        __syncthreads();
    }
#pragma unroll
    for (int k = 0; k < kTpt; ++k) {
        const int64_t t = base + threadIdx.x + k * kBlock;
        if (t >= n_tgt) continue;
        float4 v = vel[t];
        v.x = fmaf(G * ax[k], dt, v.x);
        v.y = fmaf(G * ay[k], dt, v.y);
        v.z = fmaf(G * az[k], dt, v.z);
        vel[t] = v;
        const float m = pos_src[tgt_offset + t].w;
        pos_out[t] = make_float4(fmaf(v.x, dt, xi[k]), fmaf(v.y, dt, yi[k]), fmaf(v.z, dt, zi[k]), m);
    }
}

}  // namespace

cudaError_t nbody_step_f32(const float4 *pos_src, int64_t n_src, float4 *vel, float4 *pos_out, int64_t n_tgt,
                           const jacc_nbody_params_t *p, const jacc_schedule_t *, cudaStream_t st, int *launches) {
    if (n_tgt <= 0) return cudaSuccess;
    const int64_t grid = (n_tgt + kBlock * kTpt - 1) / (kBlock * kTpt);
    nbody_kernel<<<(unsigned)grid, kBlock, 0, st>>>(pos_src, n_src, vel, pos_out, n_tgt, p->tgt_offset, p->dt,
                                                    p->eps2, p->G);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
