// FP32 pipe throughput on sm_100a: what the N-body inner loop can reach.
// Independent dependency chains (C per thread) of one instruction kind, or
// interleaved mixes, over a fixed number of iterations; every SM holds W
// warps.  Reports FP32 lane-ops per clock per SM (an FFMA2 counts 2 lane-ops
// per thread, an FFMA 1) against the nominal 128, and MUFU.RSQ per clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_pipes fp32_pipes.cu && /tmp/fp32_pipes
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }

// kind 0: FFMA2 3-reg   1: FFMA scalar 3-reg   2: FADD2   3: FMUL2
//      4: 2 FFMA2 + 1 FFMA (mix)   5: FFMA2 + FFMA alternating
//      6: 11 FFMA2 + 2 MUFU.RSQ (N-body pair-source mix)
template <int KIND, int C>
__global__ void pipe_kernel(float *out, int iters, float s) {
    float2 a[C], b[C];
    float x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        a[c] = make_float2(threadIdx.x * 1e-7f + c, c * 0.5f);
        b[c] = make_float2(1.0000001f, 0.9999999f);
        x[c] = threadIdx.x * 1e-6f + c;
    }
    const float2 s2 = make_float2(s, s * 0.5f);
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (KIND == 0) a[c] = ffma2(a[c], b[c], s2);
            if (KIND == 1) x[c] = fmaf(x[c], b[c].x, s2.y);
            if (KIND == 2) a[c] = __fadd2_rn(a[c], b[c]);
            if (KIND == 3) a[c] = __fmul2_rn(a[c], b[c]);
            if (KIND == 4) {
                a[c] = ffma2(a[c], b[c], s2);
                b[c] = ffma2(b[c], s2, a[c]);
                x[c] = fmaf(x[c], a[c].y, b[c].x);
            }
            if (KIND == 5) {
                a[c] = ffma2(a[c], b[c], s2);
                x[c] = fmaf(x[c], b[c].y, s2.x);
            }
            if (KIND == 6) {
                float2 r = ffma2(a[c], a[c], s2);
                r = ffma2(b[c], b[c], r);
                r = ffma2(a[c], b[c], r);
                float2 q;
                asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(q.x) : "f"(r.x));
                asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(q.y) : "f"(r.y));
                float2 q3 = __fmul2_rn(__fmul2_rn(q, q), q);
                a[c] = ffma2(a[c], q3, a[c]);
                b[c] = ffma2(b[c], q3, b[c]);
                float2 t = ffma2(a[c], q3, b[c]);
                a[c] = __fadd2_rn(a[c], s2);
                b[c] = __fadd2_rn(b[c], t);
                t = __fadd2_rn(t, s2);
                b[c] = ffma2(t, q3, b[c]);
            }
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) acc += a[c].x + a[c].y + b[c].x + x[c];
    if (acc == 1.2345f) out[threadIdx.x] = acc;
}

template <int KIND, int C>
void run(const char *name, double lane_ops_per_chain_iter, int warps_per_sm, int sms, float *out) {
    const int block = 32 * warps_per_sm;   // one block per SM
    const int iters = 1 << 14;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    pipe_kernel<KIND, C><<<sms, block>>>(out, 16, 1e-9f);
    cudaEventRecord(e0);
    pipe_kernel<KIND, C><<<sms, block>>>(out, iters, 1e-9f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int khz;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double clocks = ms * 1e-3 * khz * 1e3;
    const double ops_per_sm = (double)block * iters * C * lane_ops_per_chain_iter;
    printf("{\"kind\": \"%s\", \"chains\": %d, \"warps_per_sm\": %d, \"ms\": %.3f, \"lane_ops_per_clk_sm\": %.1f}\n", name,
           C, warps_per_sm, ms, ops_per_sm / clocks);
}

int main() {
    float *out;
    cudaMalloc(&out, 4096 * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int w : {4, 8, 12, 16}) {
        run<0, 8>("ffma2", 2, w, sms, out);
        run<1, 8>("ffma", 1, w, sms, out);
        run<2, 8>("fadd2", 2, w, sms, out);
        run<3, 8>("fmul2", 2, w, sms, out);
        run<4, 4>("2 ffma2 + 1 ffma", 5, w, sms, out);
        run<5, 8>("ffma2 + ffma", 3, w, sms, out);
        run<6, 2>("nbody mix: 11 paired + 2 mufu (paired lane-ops)", 22, w, sms, out);
        run<6, 4>("nbody mix: 11 paired + 2 mufu (paired lane-ops)", 22, w, sms, out);
        run<6, 6>("nbody mix: 11 paired + 2 mufu (paired lane-ops)", 22, w, sms, out);
    }
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
