// common.cuh -- small device/host helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "jacc.h"
#include "kernels.h"

namespace jacc_k {

// Streaming 128-bit loads/stores: read-once data bypasses L1 allocation,
// written-once data is marked evict-first (.cs) so it does not displace
// L2-resident operands of later tasks.
__device__ __forceinline__ float4 ld_stream(const float4 *p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ int4 ld_stream(const int4 *p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(float4 *p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

inline bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// Grid for a grid-stride kernel: the advisory schedule if given,
// else enough blocks for `work_blocks` capped at `per_sm` resident blocks on
// every SM (a whole number of waves over the 148 SMs).
inline void pick_grid(const jacc_schedule_t *s, int64_t work_blocks, int per_sm, int def_block, int *grid,
                      int *block) {
    int b = def_block;
    int64_t gsz;
    if (s && s->group[0] > 0) {   // def_block is also the kernel's __launch_bounds__
        b = s->group[0];
        if (b > def_block) b = def_block;
        b = (b + 31) / 32 * 32;
    }
    if (s && s->global[0] > 0) {
        gsz = (s->global[0] + b - 1) / b;
    } else {
        int64_t cap = (int64_t)sm_count() * per_sm;
        gsz = work_blocks < cap ? work_blocks : cap;
    }
    if (gsz < 1) gsz = 1;
    if (gsz > 0x7fffffff) gsz = 0x7fffffff;
    *grid = (int)gsz;
    *block = b;
}

}  // namespace jacc_k
