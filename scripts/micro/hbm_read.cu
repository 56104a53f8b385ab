// HBM read-stream micro-benchmark (sm_100a): which load width / depth /
// grid reaches the read-only ceiling, to size the hist/reduce loaders.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_read hbm_read.cu && /tmp/hbm_read
#include <cstdio>
#include <cuda_runtime.h>

template <int D, bool W256, bool HINT>
__global__ void __launch_bounds__(256) rd(const float *__restrict__ p, size_t n, float *out) {
    constexpr int V = W256 ? 8 : 4;
    const size_t nv = n / V;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    for (; i + (D - 1) * stride < nv; i += D * stride) {
        float r[D][V];
#pragma unroll
        for (int d = 0; d < D; ++d) {
            const float *q = p + (i + d * stride) * V;
            if (W256) {
                if (HINT)
                    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=f"(r[d][0]), "=f"(r[d][1]), "=f"(r[d][2]), "=f"(r[d][3]), "=f"(r[d][4]),
                                   "=f"(r[d][5]), "=f"(r[d][6]), "=f"(r[d][7]) : "l"(q));
                else
                    asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                 : "=f"(r[d][0]), "=f"(r[d][1]), "=f"(r[d][2]), "=f"(r[d][3]), "=f"(r[d][4]),
                                   "=f"(r[d][5]), "=f"(r[d][6]), "=f"(r[d][7]) : "l"(q));
            } else {
                if (HINT)
                    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(r[d][0]), "=f"(r[d][1]), "=f"(r[d][2]), "=f"(r[d][3]) : "l"(q));
                else
                    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                                 : "=f"(r[d][0]), "=f"(r[d][1]), "=f"(r[d][2]), "=f"(r[d][3]) : "l"(q));
            }
        }
#pragma unroll
        for (int d = 0; d < D; ++d)
#pragma unroll
            for (int v = 0; v < V; ++v) acc += r[d][v];
    }
    for (; i < nv; i += stride)   // tail: one vector at a time
#pragma unroll
        for (int v = 0; v < V; ++v) acc += p[i * V + v];
    if (acc == 1234.5f) out[0] = acc;   // keep the loads alive
}

template <int D, bool W256, bool HINT>
void run(const char *name, const float *p, size_t n, float *out, int blocks_per_sm, int sms, float *flush,
         size_t flush_n) {
    const int grid = blocks_per_sm * sms;
    float best = 1e30f;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int r = 0; r < 6; ++r) {
        cudaMemsetAsync(flush, r, flush_n * 4);   // evict L2
        cudaEventRecord(e0);
        rd<D, W256, HINT><<<grid, 256>>>(p, n, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (r > 0 && ms < best) best = ms;
    }
    printf("{\"kernel\": \"%s\", \"depth\": %d, \"blocks_per_sm\": %d, \"us\": %.1f, \"GB/s\": %.0f}\n", name, D,
           blocks_per_sm, best * 1e3, n * 4.0 / (best * 1e-3) / 1e9);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t n = (size_t)1 << 28;   // 1 GiB
    const size_t fn = (size_t)64 << 20;
    float *p, *out, *flush;
    cudaMalloc(&p, n * 4); cudaMalloc(&out, 64); cudaMalloc(&flush, fn * 4);
    cudaMemset(p, 0, n * 4);
    for (int b : {4, 8}) {
        run<2, false, false>("v4", p, n, out, b, sms, flush, fn);
        run<4, false, false>("v4", p, n, out, b, sms, flush, fn);
        run<8, false, false>("v4", p, n, out, b, sms, flush, fn);
        run<4, false, true>("v4+L2::256B", p, n, out, b, sms, flush, fn);
        run<2, true, false>("v8", p, n, out, b, sms, flush, fn);
        run<4, true, false>("v8", p, n, out, b, sms, flush, fn);
        run<2, true, true>("v8+L2::256B", p, n, out, b, sms, flush, fn);
        run<4, true, true>("v8+L2::256B", p, n, out, b, sms, flush, fn);
    }
    printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
