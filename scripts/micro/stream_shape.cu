// HBM stream shapes (sm_100a): which store flavour / vector width / depth
// reaches the highest rate for a given read:write mix -- to size the
// Black-Scholes (1 read : 2 writes) and histogram (read only) loaders.
// Variants: store .cs (evict-first) vs default write-back vs .L1::no_allocate;
// 128-bit vs 256-bit (v8) accesses; D vectors in flight per stream; 256- or
// 512-thread blocks.  L2 flushed (written then read) before every launch;
// CUDA events; 2^26 floats per stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_shape stream_shape.cu && /tmp/stream_shape
#include <cstdio>
#include <cuda_runtime.h>

struct f8 { float v[8]; };

template <bool V8>
__device__ __forceinline__ void ld(const float *p, float *r) {
    if (V8)
        asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                     : "l"(p));
    else
        asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]) : "l"(p));
}
// S: 0 = .cs, 1 = default (wb), 2 = .L1::no_allocate, 3 = .L2::evict_first via .cs on v8
template <bool V8, int S>
__device__ __forceinline__ void st(float *p, const float *r) {
    if (V8) {
        if (S == 0)
            asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]),
                         "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
        else if (S == 1)
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]),
                         "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
        else
            asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r[0]),
                         "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]) : "memory");
    } else {
        if (S == 0)
            asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3])
                         : "memory");
        else if (S == 1)
            asm volatile("st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3])
                         : "memory");
        else
            asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(r[0]), "f"(r[1]),
                         "f"(r[2]), "f"(r[3]) : "memory");
    }
}

template <int R, int W, bool V8, int S, int D>
__global__ void __launch_bounds__(512) mix(const float *__restrict__ a, float *__restrict__ c, float *__restrict__ d,
                                           size_t n, float *sink) {
    constexpr int V = V8 ? 8 : 4;
    const size_t nv = n / V;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += D * stride) {
        float x[D][8];
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const size_t j = i + k * stride;
            if (R >= 1 && j < nv) ld<V8>(a + j * V, x[k]);
            else
#pragma unroll
                for (int e = 0; e < 8; ++e) x[k][e] = 1.f;
        }
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const size_t j = i + k * stride;
            if (j >= nv) break;
            if (W >= 1) st<V8, S>(c + j * V, x[k]);
            if (W >= 2) {
                float y[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) y[e] = x[k][e] * 2.f;
                st<V8, S>(d + j * V, y);
            }
            if (W == 0)
#pragma unroll
                for (int e = 0; e < V; ++e) acc += x[k][e];
        }
    }
    if (W == 0 && acc == 123.456f) *sink = acc;
}

__global__ void flush_read(const float4 *p, size_t n4, float *sink) {
    float acc = 0.f;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        acc += p[i].x;
    if (acc == 123.456f) *sink = acc;
}

template <int R, int W, bool V8, int S, int D>
void run(const char *tag, int block, int per_sm, float *a, float *c, float *d, size_t n, float *sink, char *fl,
         size_t flb, int sms) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * per_sm;
    float sum = 0.f, best = 1e30f;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
        cudaMemset(fl, r, flb);
        flush_read<<<sms * 4, 512>>>((const float4 *)fl, flb / 16, sink);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        mix<R, W, V8, S, D><<<grid, block>>>(a, c, d, n, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2) { sum += ms; if (ms < best) best = ms; }
    }
    const double bytes = (double)n * 4 * (R + W);
    printf("{\"R\": %d, \"W\": %d, \"v8\": %d, \"store\": \"%s\", \"D\": %d, \"block\": %d, \"per_sm\": %d, "
           "\"mean_us\": %.2f, \"mean_GBps\": %.1f, \"best_GBps\": %.1f, \"err\": \"%s\"}\n",
           R, W, (int)V8, S == 0 ? "cs" : S == 1 ? "wb" : "L1na", D, block, per_sm, sum / reps * 1e3,
           bytes / (sum / reps * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    (void)tag;
}

int main() {
    const size_t n = (size_t)1 << 26;
    float *a, *c, *d, *sink;
    char *fl;
    const size_t flb = (size_t)256 << 20;
    cudaMalloc(&a, n * 4); cudaMalloc(&c, n * 4); cudaMalloc(&d, n * 4);
    cudaMalloc(&fl, flb); cudaMalloc(&sink, 4);
    cudaMemset(a, 0, n * 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // 1 read : 2 writes (Black-Scholes)
    run<1, 2, false, 0, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, false, 1, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, false, 2, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, true, 0, 2>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, true, 1, 2>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, true, 1, 1>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, true, 1, 4>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, false, 1, 4>("", 512, 4, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, false, 1, 2>("", 512, 4, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, false, 1, 1>("", 512, 4, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, false, 1, 1>("", 256, 16, a, c, d, n, sink, fl, flb, sms);
    run<1, 2, true, 1, 2>("", 512, 4, a, c, d, n, sink, fl, flb, sms);
    // 1 read : 1 write (copy) and write only
    run<1, 1, false, 0, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 1, false, 1, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 1, true, 1, 2>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<0, 1, false, 0, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<0, 1, false, 1, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<0, 1, true, 1, 2>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    // read only
    run<1, 0, false, 0, 3>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 0, false, 0, 4>("", 512, 4, a, c, d, n, sink, fl, flb, sms);
    run<1, 0, true, 0, 2>("", 256, 8, a, c, d, n, sink, fl, flb, sms);
    run<1, 0, true, 0, 4>("", 512, 4, a, c, d, n, sink, fl, flb, sms);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
