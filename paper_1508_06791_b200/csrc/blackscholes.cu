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

// The same arithmetic on two options at once with the sm_100 paired FP32
// instructions (FADD2 / FMUL2 / FFMA2): the FP32 work per option is
// unchanged, its issue slots are halved -- the scalar kernel is issue-bound
// (ncu: ~77 % issue-active with HBM at ~60 %).  MUFU ops stay per element.
__device__ __forceinline__ float2 F2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

__device__ __forceinline__ float2 bs_poly2(float2 t) {   // t * P(t) * 0.398942280
    constexpr double k = 0.398942280;
    const float2 c1 = F2((float)(k * 0.319381530)), c2 = F2((float)(k * -0.356563782)),
                 c3 = F2((float)(k * 1.781477937)), c4 = F2((float)(k * -1.821255978)),
                 c5 = F2((float)(k * 1.330274429));
    return mul2(t, fma2(t, fma2(t, fma2(t, fma2(t, c5, c4), c3), c2), c1));
}

__device__ __forceinline__ float2 abs2(float2 v) {   // sign bits cleared on the integer pipe (LOP3)
    return make_float2(__uint_as_float(__float_as_uint(v.x) & 0x7fffffffu),
                       __uint_as_float(__float_as_uint(v.y) & 0x7fffffffu));
}

// The APARAPI mapping computes S and K with the same FFMA of u, so they are
// the same float and ln(S/K) = 0 EXACTLY (in the oracle's fp64 as well):
//   d1 = (R + sigma^2/2) T / (sigma sqrt T)          -- no logarithm,
//   S / (K e^{-RT}) = e^{RT}                          -- no division by kexp.
// One reciprocal of q1 q2 e^{-RT} then yields 1/q1, 1/q2 and e^{RT}:
// four MUFU ops per option (rsqrt, two ex2, one rcp) instead of six --
// the MUFU pipe was 65 % busy (ncu) on the general form.
// put comes from put-call parity, call - S + K e^{-RT}: an exact identity of
// this formula (the A&S CND satisfies phi(-x) = 1 - phi(x) by construction,
// SURVEY §8(c)-B), so it is the same value up to fp32 rounding.
__device__ __forceinline__ void bs_aparapi2(float2 u, float2 &call, float2 &put) {
    const float2 m1 = F2(-1.0f), one = F2(1.0f);
    const float2 S = fma2(F2(10.0f - 100.0f), u, F2(100.0f));       // = K
    const float2 T = fma2(F2(1.0f - 10.0f), u, F2(10.0f));
    const float2 R = fma2(F2(0.01f - 0.05f), u, F2(0.05f));
    const float2 V = fma2(F2(0.01f - 0.10f), u, F2(0.10f));
    const float2 v2t = mul2(mul2(V, V), T);                                            // sigma^2 T
    const float2 rs = make_float2(rsqrtf(v2t.x), rsqrtf(v2t.y));                      // 1/(sigma sqrt T)
    const float2 sst = mul2(v2t, rs);                                                  // sigma sqrt T
    const float2 rt = mul2(R, T);
    const float2 ert = mul2(rt, F2(-1.44269504088896340736f));
    const float2 ekr = make_float2(ex2_approx(ert.x), ex2_approx(ert.y));             // e^{-RT}
    const float2 d1 = mul2(fma2(F2(0.5f), v2t, rt), rs);
    const float2 d2 = fma2(sst, m1, d1);
    const float2 q1 = fma2(F2(0.2316419f), abs2(d1), one);
    const float2 q2 = fma2(F2(0.2316419f), abs2(d2), one);
    const float2 qq = mul2(q1, q2);
    const float2 den = mul2(qq, ekr);
    const float2 rr = make_float2(__fdividef(1.0f, den.x), __fdividef(1.0f, den.y));  // 1/(q1 q2 e^{-RT})
    const float2 rq = mul2(rr, ekr);                                                   // 1/(q1 q2)
    const float2 ratio = mul2(rr, qq);                                                 // e^{RT}
    const float2 ea = mul2(mul2(F2(-0.72134752044448170368f), d1), d1);
    const float2 e1 = make_float2(ex2_approx(ea.x), ex2_approx(ea.y));                 // e^{-d1^2/2}
    const float2 e2 = mul2(e1, ratio);                                                 // e^{-d2^2/2}
    const float2 w1 = mul2(e1, bs_poly2(mul2(q2, rq)));                               // t1 = 1/q1
    const float2 w2 = mul2(e2, bs_poly2(mul2(q1, rq)));                               // t2 = 1/q2
    // phi(d1) and -phi(d2); call = S phi(d1) - K e^{-RT} phi(d2) = S (phi(d1) -
    // e^{-RT} phi(d2)) with K = S
    const float2 om1 = fma2(w1, m1, one), wm2 = add2(w2, m1);
    const float2 pd1 = make_float2(d1.x < 0.f ? w1.x : om1.x, d1.y < 0.f ? w1.y : om1.y);
    const float2 npd2 = make_float2(d2.x < 0.f ? -w2.x : wm2.x, d2.y < 0.f ? -w2.y : wm2.y);
    call = mul2(S, fma2(ekr, npd2, pd1));
    put = fma2(S, add2(ekr, m1), call);    // call - S + S e^{-RT}
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

template <int kDepth, int kMinBlocks>
__global__ void __launch_bounds__(256, kMinBlocks) bs_v4_kernel(const float4 *__restrict__ u4, float4 *__restrict__ call4,
                                                    float4 *__restrict__ put4, int64_t n4,
                                                    const float *__restrict__ ut, float *__restrict__ ct,
                                                    float *__restrict__ pt, int tail) {
    // kDepth vectors per trip; the next trip's kDepth loads are issued before
    // this trip's 4 * kDepth options are priced, so every thread always has
    // kDepth 128-bit loads in flight (the kernel is otherwise latency-bound:
    // ncu showed long-scoreboard stalls dominating with one load in flight).
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
            float2 c01, p01, c23, p23;
            bs_aparapi2(make_float2(cur[d].x, cur[d].y), c01, p01);
            bs_aparapi2(make_float2(cur[d].z, cur[d].w), c23, p23);
            st_stream(call4 + j, make_float4(c01.x, c01.y, c23.x, c23.y));
            st_stream(put4 + j, make_float4(p01.x, p01.y, p23.x, p23.y));
        }
    }
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < tail) bs_aparapi(ut[t], ct[t], pt[t]);
}

// 256-bit I/O (sm_100 LDG.256 / STG.256): 8 options per thread per trip, the
// next trip's vector loaded before this one is priced.  Measured at 2^26
// (same-box A/B, scripts/ab/ab.sh): 137.3 us vs 141.4 us for the 128-bit
// kernel above at its best depth; the plain 1-read : 2-write stream of
// scripts/micro/stream_shape.cu peaks with this shape too (256-bit, one
// vector per thread in flight: 130 us = 6.18 TB/s, vs 5.80 TB/s for 128-bit
// accesses three deep).  Default (write-back) stores: .cs measured the same.
struct f8 {
    float v[8];
};
__device__ __forceinline__ f8 ld_stream8(const float *p) {
    f8 r;
    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                   "=f"(r.v[7])
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st8(float *p, const f8 &r) {
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]),
                 "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}

__global__ void __launch_bounds__(256, 4) bs_v8_kernel(const float *__restrict__ u, float *__restrict__ call,
                                                       float *__restrict__ put, int64_t n8, const float *__restrict__ ut,
                                                       float *__restrict__ ct, float *__restrict__ pt, int tail) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    f8 nxt;
    if (i < n8) nxt = ld_stream8(u + 8 * i);
    for (; i < n8; i += stride) {
        const f8 cur = nxt;
        if (i + stride < n8) nxt = ld_stream8(u + 8 * (i + stride));
        f8 c, p;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            float2 cc, pp;
            bs_aparapi2(make_float2(cur.v[2 * h], cur.v[2 * h + 1]), cc, pp);
            c.v[2 * h] = cc.x;
            c.v[2 * h + 1] = cc.y;
            p.v[2 * h] = pp.x;
            p.v[2 * h + 1] = pp.y;
        }
        st8(call + 8 * i, c);
        st8(put + 8 * i, p);
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
    if ((((uintptr_t)u | (uintptr_t)call | (uintptr_t)put) & 31) == 0) {   // 256-bit accesses
        const int64_t n8 = n / 8;
        pick_grid(s, (n8 + 255) / 256, 8, 256, &grid, &block);
        bs_v8_kernel<<<grid, block, 0, st>>>(u, call, put, n8, u + 8 * n8, call + 8 * n8, put + 8 * n8,
                                             (int)(n - 8 * n8));
    } else if (aligned16(u) && aligned16(call) && aligned16(put)) {
        const int64_t n4 = n / 4;
        // (A TMA-staged variant -- cp.async.bulk into a 4-stage mbarrier ring,
        // 8 consumer warps -- measured 163 us vs 155 us for this one: the
        // kernel is issue-bound once two loads per thread are in flight.)
        // 3 vectors in flight per thread, 3 blocks per SM (80 registers):
        // measured 146 us vs 149 (2, 4 blocks), 149 (4, 2), 167 (2, 1).  The
        // grid asks for 8 blocks per SM (2.7 waves of the grid-stride loop):
        // exactly one resident wave (148 x 3) measured slower, 146 vs 139 us.
        // (re-measured with the 4-MUFU form: depth/blocks 3/3 137-142 us,
        // 3/4 (16 B spills) 138-145, 2/4 142-145, 4/3 140-146)
        pick_grid(s, (n4 + 255) / 256, 8, 256, &grid, &block);
        bs_v4_kernel<3, 3><<<grid, block, 0, st>>>((const float4 *)u, (float4 *)call, (float4 *)put, n4, u + 4 * n4,
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
