// HBM stream ceilings by read/write mix (sm_100a): what a plain copy-like
// kernel reaches when it reads R and writes W 16-byte vectors per element
// group -- the memory roof of each HBM-bound task's own mix:
//   R1W0 reduce / histogram (read only)   R2W1 vadd (8 B read, 4 B written)
//   R1W2 Black-Scholes (4 B read, 8 B written)
// Same loader shape as the product kernels: grid-stride 128-bit loads, 3
// vectors in flight per stream, streaming stores (.cs), 256 threads, 8
// blocks per SM requested.  L2 flushed (256 MiB written then read) before
// every launch; CUDA events; 2^26 elements per stream (256 MiB each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_mix stream_mix.cu && /tmp/stream_mix
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float4 ldv(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void stv(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

template <int R, int W>
__global__ void __launch_bounds__(256) mix(const float4 *__restrict__ a, const float4 *__restrict__ b,
                                           float4 *__restrict__ c, float4 *__restrict__ d, size_t n4,
                                           float *sink) {
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    float acc = 0.f;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += 3 * stride) {
        float4 x[3], y[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const size_t j = i + k * stride;
            x[k] = (R >= 1 && j < n4) ? ldv(a + j) : make_float4(1.f, 2.f, 3.f, 4.f);
            y[k] = (R >= 2 && j < n4) ? ldv(b + j) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const size_t j = i + k * stride;
            if (j >= n4) break;
            const float4 s = make_float4(x[k].x + y[k].x, x[k].y + y[k].y, x[k].z + y[k].z, x[k].w + y[k].w);
            if (W >= 1) stv(c + j, s);
            if (W >= 2) stv(d + j, x[k]);
            if (W == 0) acc += s.x + s.y + s.z + s.w;
        }
    }
    if (W == 0 && acc == 123.456f) *sink = acc;
}

template <int R, int W>
void run(const char *name, float4 *a, float4 *b, float4 *c, float4 *d, size_t n4, float *sink, char *fl,
         size_t flb, int grid) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f, sum = 0.f;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
        cudaMemset(fl, r, flb);   // evict L2: write, then read (clean lines)
        mix<1, 0><<<grid, 256>>>((const float4 *)fl, nullptr, nullptr, nullptr, flb / 16, sink);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        mix<R, W><<<grid, 256>>>(a, b, c, d, n4, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2) {
            sum += ms;
            if (ms < best) best = ms;
        }
    }
    const double bytes = (double)n4 * 16 * (R + W);
    printf("{\"mix\": \"%s\", \"reads\": %d, \"writes\": %d, \"mean_us\": %.2f, \"mean_GBps\": %.1f, \"best_GBps\": %.1f}\n",
           name, R, W, sum / reps * 1e3, bytes / (sum / reps * 1e-3) / 1e9, bytes / (best * 1e-3) / 1e9);
}

int main() {
    const size_t n4 = (size_t)1 << 24;   // 2^26 floats per stream
    float4 *a, *b, *c, *d;
    char *fl;
    float *sink;
    const size_t flb = (size_t)256 << 20;
    cudaMalloc(&a, n4 * 16); cudaMalloc(&b, n4 * 16); cudaMalloc(&c, n4 * 16); cudaMalloc(&d, n4 * 16);
    cudaMalloc(&fl, flb); cudaMalloc(&sink, 4);
    cudaMemset(a, 0, n4 * 16); cudaMemset(b, 0, n4 * 16);
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = sms * 8;
    run<1, 0>("read only (reduce, histogram)", a, b, c, d, n4, sink, fl, flb, grid);
    run<2, 1>("2 reads : 1 write (vadd)", a, b, c, d, n4, sink, fl, flb, grid);
    run<1, 1>("1 read : 1 write (copy)", a, b, c, d, n4, sink, fl, flb, grid);
    run<1, 2>("1 read : 2 writes (Black-Scholes)", a, b, c, d, n4, sink, fl, flb, grid);
    run<0, 1>("write only", a, b, c, d, n4, sink, fl, flb, grid);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
