// vadd.cu -- Vector Addition (§4.2): c[i] = a[i] + b[i].
//
// An elementwise map: each element is touched once, so the kernel is pure
// HBM streaming at 12 algorithmic bytes per element (read a, b; write c).
// sm_100a design: grid-stride over 128-bit vectors (ld.global.nc.L1::
// no_allocate / st.global.cs), 4 independent vectors in flight per operand
// per thread, grid = 8 resident 256-thread blocks on each of the 148 SMs;
// from 2^26 elements (32-byte aligned) 256-bit vectors, 2 in flight.
// The iteration space maps onto threads as the @Jacc(ONE_DIMENSION) model
// says; fewer threads than elements is the block-cyclic mapping
// of P:163-164 (reading R15): any schedule gives the same bits.
#include "common.cuh"
#include "kernels.h"

namespace jacc_k {
namespace {

constexpr int kUnroll = 4;

__global__ void __launch_bounds__(256) vadd_v4_kernel(const float4 *__restrict__ a, const float4 *__restrict__ b,
                                                      float4 *__restrict__ c, int64_t n4,
                                                      const float *__restrict__ at, const float *__restrict__ bt,
                                                      float *__restrict__ ct, int tail) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (kUnroll - 1) * stride < n4; i += kUnroll * stride) {
        float4 x[kUnroll], y[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            x[u] = ld_stream(a + i + u * stride);
            y[u] = ld_stream(b + i + u * stride);
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            st_stream(c + i + u * stride, make_float4(x[u].x + y[u].x, x[u].y + y[u].y, x[u].z + y[u].z,
                                                      x[u].w + y[u].w));
    }
    if (i < n4) {   // the remainder (< kUnroll vectors): loads issued together
        float4 x[kUnroll - 1], y[kUnroll - 1];
#pragma unroll
        for (int u = 0; u < kUnroll - 1; ++u)
            if (i + u * stride < n4) {
                x[u] = ld_stream(a + i + u * stride);
                y[u] = ld_stream(b + i + u * stride);
            }
#pragma unroll
        for (int u = 0; u < kUnroll - 1; ++u)
            if (i + u * stride < n4)
                st_stream(c + i + u * stride,
                          make_float4(x[u].x + y[u].x, x[u].y + y[u].y, x[u].z + y[u].z, x[u].w + y[u].w));
    }
    // the (< 4) trailing scalars
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < tail) ct[t] = at[t] + bt[t];
}


// 256-bit form (sm_100 LDG/STG .ENL2.256) for large, 32-byte aligned
// operands: 2 vectors of 8 per operand per thread in flight.  Same-box A/B
// (scripts/ab/ab.sh, kbench vadd): 2^28 502 -> 477 us (6.76 TB/s); at 2^24 the
// 128-bit kernel stays ahead (31.4 vs 32.2 us), hence the size threshold.
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
__device__ __forceinline__ void st_stream8(float *p, const f8 &r) {
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]),
                 "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
                 : "memory");
}
constexpr int kDepth8 = 2;
constexpr int64_t kMinN8 = (int64_t)1 << 26;   // elements: the 256-bit form from here on

__global__ void __launch_bounds__(256) vadd_v8_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                                      float *__restrict__ c, int64_t n8, int tail) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += kDepth8 * stride) {
        f8 x[kDepth8], y[kDepth8];
#pragma unroll
        for (int u = 0; u < kDepth8; ++u)
            if (i + u * stride < n8) {
                x[u] = ld_stream8(a + 8 * (i + u * stride));
                y[u] = ld_stream8(b + 8 * (i + u * stride));
            }
#pragma unroll
        for (int u = 0; u < kDepth8; ++u)
            if (i + u * stride < n8) {
                f8 z;
#pragma unroll
                for (int e = 0; e < 8; ++e) z.v[e] = x[u].v[e] + y[u].v[e];
                st_stream8(c + 8 * (i + u * stride), z);
            }
    }
    // the (< 8) trailing scalars
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < tail) c[8 * n8 + t] = a[8 * n8 + t] + b[8 * n8 + t];
}

__global__ void __launch_bounds__(256) vadd_scalar_kernel(const float *__restrict__ a, const float *__restrict__ b,
                                                          float *__restrict__ c, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) c[i] = a[i] + b[i];
}

}  // namespace

cudaError_t vadd_f32(const float *a, const float *b, float *c, int64_t n, const jacc_schedule_t *s, cudaStream_t st,
                     int *launches) {
    if (n <= 0) return cudaSuccess;
    int grid, block;
    if (n >= kMinN8 && (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 31) == 0) {
        const int64_t n8 = n / 8;
        pick_grid(s, (n8 + 255) / 256, 8, 256, &grid, &block);
        vadd_v8_kernel<<<grid, block, 0, st>>>(a, b, c, n8, (int)(n - 8 * n8));
    } else if (aligned16(a) && aligned16(b) && aligned16(c)) {
        const int64_t n4 = n / 4;
        const int tail = (int)(n - 4 * n4);
        // 8 blocks per SM requested although 5 are resident (42 registers):
        // the grid-stride loop over 1.6 waves measured faster than exactly
        // one resident wave (2^28: 505 vs 515 us)
        pick_grid(s, (n4 + 255) / 256, 8, 256, &grid, &block);
        vadd_v4_kernel<<<grid, block, 0, st>>>((const float4 *)a, (const float4 *)b, (float4 *)c, n4, a + 4 * n4,
                                               b + 4 * n4, c + 4 * n4, tail);
    } else {
        pick_grid(s, (n + 255) / 256, 8, 256, &grid, &block);
        vadd_scalar_kernel<<<grid, block, 0, st>>>(a, b, c, n);
    }
    ++*launches;
    return cudaGetLastError();
}

}  // namespace jacc_k
