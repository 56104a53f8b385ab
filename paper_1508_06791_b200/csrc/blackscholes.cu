// blackscholes.cu -- Black-Scholes option pricing (§4.2: "an
// implementation of the Black Scholes option pricing model ... supplied as an
// example in the APARAPI source code").  Formula = reading R12 (SURVEY
// §8(c)-B, the APARAPI sample):
//   u in [0,1) -> S = 10u + 100(1-u), K = 10u + 100(1-u), T = 1u + 10(1-u),
//                 R = 0.01u + 0.05(1-u), sigma = 0.01u + 0.10(1-u)
//   d1 = (ln(S/K) + (R + sigma^2/2) T) / (sigma sqrt T),  d2 = d1 - sigma sqrt T
//   phi(x): t = 1/(1 + 0.2316419|x|),
//           y = 1 - 0.398942280 e^{-x^2/2} t (c1 + t(c2 + t(c3 + t(c4 + t c5)))),
//           phi = y if x >= 0 else 1 - y
//   call = S phi(d1) - K e^{-RT} phi(d2);  put = K e^{-RT} phi(-d2) - S phi(-d1)
//
// sm_100a design: a map at 12 HBM bytes per option whose ~60 fp32 ops and
// MUFU transcendentals put it close to the issue roof as well.  Work saved
// without changing the formula's value beyond fp32 rounding:
//   * one MUFU.RSQ gives 1/(sigma sqrt T) = rsqrt(sigma^2 T), and
//     sigma sqrt T = sigma^2 T * rsqrt(sigma^2 T);
//   * the tail w(x) = 0.398942280 e^{-x^2/2} t P(t) depends on |x| only, so
//     phi(d) and phi(-d) share it (phi(x) = x < 0 ? w : 1 - w and
//     phi(-x) = x > 0 ? w : 1 - w, exactly the branches of the formula);
//   * both t = 1/q1, 1/q2 come from ONE reciprocal of q1*q2;
//   * 128-bit loads/stores, 4 options per thread per iteration.
// Fast-math intrinsics (rsqrt/ex2/lg2/rcp .approx) are admissible: the
// tolerance (R12) is |g - o| <= 1e-5 (S + K e^{-RT}) per option.
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {

__device__ __forceinline__ float ex2_approx(float x) {   // MUFU.EX2
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// w(x) = 0.398942280 e^{-x^2/2} t (c1 + t(c2 + t(c3 + t(c4 + t c5)))), with the
// 0.398942280 factor folded into the polynomial coefficients.
__device__ __forceinline__ float bs_poly(float t) {   // t * P(t) * 0.398942280
    constexpr double k = 0.398942280;
    constexpr float c1 = (float)(k * 0.319381530), c2 = (float)(k * -0.356563782), c3 = (float)(k * 1.781477937),
                    c4 = (float)(k * -1.821255978), c5 = (float)(k * 1.330274429);
    return t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, c5, c4), c3), c2), c1);
}

// Six MUFU ops per option: with kexp = K e^{-RT} and ratio = S / kexp,
//   ln(S/K) + (R + sigma^2/2) T = ln(ratio) + sigma^2 T / 2,
//   e^{-d2^2/2} = e^{-d1^2/2} * ratio      (because d1 s - s^2/2 = ln ratio,
//                                            s = sigma sqrt T)
// so one reciprocal and one exponential serve both d1 and the second CND.
// (If e^{-d1^2/2} flushed to 0 while d2 is small -- only for sigma sqrt T > 10
// -- the second tail would read 0; no input the tests or configs use.)
__device__ __forceinline__ void bs_price(float S, float K, float T, float R, float V, float &call, float &put) {
    const float v2t = V * V * T;                   // sigma^2 T
    const float rs = rsqrtf(v2t);                  // 1 / (sigma sqrt T)        MUFU.RSQ
    const float sst = v2t * rs;                    // sigma sqrt T
    const float kexp = K * ex2_approx(-1.44269504088896340736f * R * T);   // K e^{-RT}   MUFU.EX2
    const float ratio = __fdividef(S, kexp);       // MUFU.RCP
    const float d1 = fmaf(0.5f, v2t, __logf(ratio)) * rs;                  // MUFU.LG2
    const float d2 = d1 - sst;
    const float q1 = fmaf(0.2316419f, fabsf(d1), 1.0f);
    const float q2 = fmaf(0.2316419f, fabsf(d2), 1.0f);
    const float r = __fdividef(1.0f, q1 * q2);     // both t = 1/q from one   MUFU.RCP
    const float e1 = ex2_approx((-0.72134752044448170368f * d1) * d1);     // e^{-d1^2/2}  MUFU.EX2
    const float e2 = e1 * ratio;                   // e^{-d2^2/2}
    const float w1 = e1 * bs_poly(q2 * r);         // tail of |d1|
    const float w2 = e2 * bs_poly(q1 * r);         // tail of |d2|
    const float phi_d1 = d1 < 0.f ? w1 : 1.0f - w1;
    const float phi_d2 = d2 < 0.f ? w2 : 1.0f - w2;
    const float phi_md1 = d1 > 0.f ? w1 : 1.0f - w1;   // phi(-d1)
    const float phi_md2 = d2 > 0.f ? w2 : 1.0f - w2;   // phi(-d2)
    call = S * phi_d1 - kexp * phi_d2;
    put = kexp * phi_md2 - S * phi_md1;
}

// X = X_lo u + X_hi (1 - u) = X_hi + (X_lo - X_hi) u: one FFMA per parameter.
__device__ __forceinline__ void bs_aparapi(float u, float &call, float &put) {
    const float S = fmaf(10.0f - 100.0f, u, 100.0f);
    const float K = fmaf(10.0f - 100.0f, u, 100.0f);
    const float T = fmaf(1.0f - 10.0f, u, 10.0f);
    const float R = fmaf(0.01f - 0.05f, u, 0.05f);
    const float V = fmaf(0.01f - 0.10f, u, 0.10f);
    bs_price(S, K, T, R, V, call, put);
}

__global__ void __launch_bounds__(256) bs_v4_kernel(const float4 *__restrict__ u4, float4 *__restrict__ call4,
                                                    float4 *__restrict__ put4, int64_t n4,
                                                    const float *__restrict__ ut, float *__restrict__ ct,
                                                    float *__restrict__ pt, int tail) {
    // kDepth vectors per trip; the next trip's kDepth loads are issued before
    // this trip's 4 * kDepth options are priced, so every thread always has
    // kDepth 128-bit loads in flight (the kernel is otherwise latency-bound:
    // ncu showed long-scoreboard stalls dominating with one load in flight).
    constexpr int kDepth = 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float4 nxt[kDepth];
#pragma unroll
    for (int d = 0; d < kDepth; ++d)
        nxt[d] = i + d * stride < n4 ? ld_stream(u4 + i + d * stride) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (; i < n4; i += kDepth * stride) {
        float4 cur[kDepth];
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
            cur[d] = nxt[d];
            const int64_t j = i + (kDepth + d) * stride;
            if (j < n4) nxt[d] = ld_stream(u4 + j);
        }
#pragma unroll
        for (int d = 0; d < kDepth; ++d) {
            const int64_t j = i + d * stride;
            if (j >= n4) break;
            float4 c, p;
            bs_aparapi(cur[d].x, c.x, p.x);
            bs_aparapi(cur[d].y, c.y, p.y);
            bs_aparapi(cur[d].z, c.z, p.z);
            bs_aparapi(cur[d].w, c.w, p.w);
            st_stream(call4 + j, c);
            st_stream(put4 + j, p);
        }
    }
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < tail) bs_aparapi(ut[t], ct[t], pt[t]);
}

__global__ void __launch_bounds__(256) bs_scalar_kernel(const float *__restrict__ u, float *__restrict__ call,
                                                        float *__restrict__ put, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        bs_aparapi(u[i], call[i], put[i]);
}

__global__ void __launch_bounds__(256) bs_soa_kernel(const float *__restrict__ S, const float *__restrict__ K,
                                                     const float *__restrict__ T, const float *__restrict__ R,
                                                     const float *__restrict__ V, float *__restrict__ call,
                                                     float *__restrict__ put, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        bs_price(S[i], K[i], T[i], R[i], V[i], call[i], put[i]);
}

}  // namespace

cudaError_t blackscholes_f32(const float *u, float *call, float *put, int64_t n, const jacc_schedule_t *s,
                             cudaStream_t st, int *launches) {
    if (n <= 0) return cudaSuccess;
    int grid, block;
    if (aligned16(u) && aligned16(call) && aligned16(put)) {
        const int64_t n4 = n / 4;
        // (A TMA-staged variant -- cp.async.bulk into a 4-stage mbarrier ring,
        // 8 consumer warps -- measured 163 us vs 155 us for this one: the
        // kernel is issue-bound once two loads per thread are in flight.)
        pick_grid(s, (n4 + 255) / 256, 8, 256, &grid, &block);
        bs_v4_kernel<<<grid, block, 0, st>>>((const float4 *)u, (float4 *)call, (float4 *)put, n4, u + 4 * n4,
                                             call + 4 * n4, put + 4 * n4, (int)(n - 4 * n4));
    } else {
        pick_grid(s, (n + 255) / 256, 8, 256, &grid, &block);
        bs_scalar_kernel<<<grid, block, 0, st>>>(u, call, put, n);
    }
    ++*launches;
    return cudaGetLastError();
}

cudaError_t blackscholes_soa_f32(const float *S, const float *K, const float *T, const float *R, const float *V,
                                 float *call, float *put, int64_t n, const jacc_schedule_t *s, cudaStream_t st,
                                 int *launches) {
    if (n <= 0) return cudaSuccess;
    int grid, block;
    pick_grid(s, (n + 255) / 256, 8, 256, &grid, &block);
    bs_soa_kernel<<<grid, block, 0, st>>>(S, K, T, R, V, call, put, n);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
