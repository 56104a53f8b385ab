// FP32 pipe micro-benchmark (sm_100a): lane-op throughput per SM per clock
// of scalar and paired FP32 instructions, alone and interleaved, to decide
// how the N-body inner loop should mix them.  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_pipes fp32_pipes.cu && /tmp/fp32_pipes
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kIters = 2048;
constexpr int kChains = 8;

enum Op { FFMA, FFMA2, FADD, FADD2, FMUL, FMUL2, MIX_FFMA2_FADD, MIX_FFMA2_FMUL, MIX_FFMA2_FFMA, MIX_FFMA2_FFMA_IMM,
          FFMA_IMM, MIX_FADD2_FMUL2_FFMA2 };

template <int OP>
__global__ void __launch_bounds__(256) kern(const float *in, float *out) {
    float2 b2 = make_float2(in[threadIdx.x & 7], in[(threadIdx.x + 1) & 7]);
    float2 c2 = make_float2(in[(threadIdx.x + 2) & 7], in[(threadIdx.x + 3) & 7]);
    float b = b2.x, c = c2.x;
    float2 a[kChains];
    float s[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) { a[i] = make_float2(in[i], in[i + 8]); s[i] = in[i + 16]; }
#pragma unroll 4
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) {
            if (OP == FFMA) { s[i] = fmaf(s[i], b, c); a[i].x = fmaf(a[i].x, b, c); }
            if (OP == FFMA_IMM) { s[i] = fmaf(s[i], b, 0.999f); a[i].x = fmaf(a[i].x, b, 1.001f); }
            if (OP == FFMA2) a[i] = __ffma2_rn(a[i], b2, c2);
            if (OP == FADD) { s[i] = s[i] + b; a[i].x = a[i].x + c; }
            if (OP == FADD2) a[i] = __fadd2_rn(a[i], b2);
            if (OP == FMUL) { s[i] = s[i] * b; a[i].x = a[i].x * c; }
            if (OP == FMUL2) a[i] = __fmul2_rn(a[i], b2);
            if (OP == MIX_FFMA2_FADD) { a[i] = __ffma2_rn(a[i], b2, c2); s[i] = s[i] + b; }
            if (OP == MIX_FFMA2_FMUL) { a[i] = __ffma2_rn(a[i], b2, c2); s[i] = s[i] * b; }
            if (OP == MIX_FFMA2_FFMA) { a[i] = __ffma2_rn(a[i], b2, c2); s[i] = fmaf(s[i], b, c); }
            if (OP == MIX_FFMA2_FFMA_IMM) { a[i] = __ffma2_rn(a[i], b2, c2); s[i] = fmaf(s[i], b, 0.999f); }
            if (OP == MIX_FADD2_FMUL2_FFMA2) {
                if (i % 3 == 0) a[i] = __fadd2_rn(a[i], b2);
                else if (i % 3 == 1) a[i] = __fmul2_rn(a[i], b2);
                else a[i] = __ffma2_rn(a[i], b2, c2);
            }
        }
    }
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < kChains; ++i) r += a[i].x + a[i].y + s[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

// lane-ops per iteration per thread (a paired op = 2 lane-ops)
static double lane_ops(int op) {
    switch (op) {
        case FFMA: case FFMA_IMM: case FADD: case FMUL: return 2.0 * kChains;
        case FFMA2: case FADD2: case FMUL2: case MIX_FADD2_FMUL2_FFMA2: return 2.0 * kChains;
        default: return 3.0 * kChains;   // mixes: paired (2) + scalar (1)
    }
}

template <int OP>
void run(const char *name, const float *in, float *out, int sms, int blocks_per_sm, int clock_khz) {
    dim3 grid(sms * blocks_per_sm);
    kern<OP><<<grid, 256>>>(in, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) kern<OP><<<grid, 256>>>(in, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = lane_ops(OP) * kIters * 256.0 * grid.x * reps;
    const double per_clk_sm = ops / (ms * 1e-3) / sms / (clock_khz * 1e3);
    printf("{\"op\": \"%s\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"lane_ops_per_clk_per_sm_at_max_clock\": %.1f}\n", name,
           blocks_per_sm, ms / reps, per_clk_sm);
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float *in, *out;
    cudaMalloc(&in, 64 * 4); cudaMalloc(&out, (size_t)p.multiProcessorCount * 8 * 256 * 4);
    float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1.0f + i * 1e-3f;
    cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
    const int S = p.multiProcessorCount;
    for (int bps : {4, 8}) {
        run<FFMA>("FFMA", in, out, S, bps, clk);
        run<FFMA_IMM>("FFMA_imm", in, out, S, bps, clk);
        run<FFMA2>("FFMA2", in, out, S, bps, clk);
        run<FADD>("FADD", in, out, S, bps, clk);
        run<FADD2>("FADD2", in, out, S, bps, clk);
        run<FMUL>("FMUL", in, out, S, bps, clk);
        run<FMUL2>("FMUL2", in, out, S, bps, clk);
        run<MIX_FFMA2_FADD>("FFMA2+FADD", in, out, S, bps, clk);
        run<MIX_FFMA2_FMUL>("FFMA2+FMUL", in, out, S, bps, clk);
        run<MIX_FFMA2_FFMA>("FFMA2+FFMA", in, out, S, bps, clk);
        run<MIX_FFMA2_FFMA_IMM>("FFMA2+FFMA_imm", in, out, S, bps, clk);
        run<MIX_FADD2_FMUL2_FFMA2>("FADD2/FMUL2/FFMA2", in, out, S, bps, clk);
    }
    printf("{\"sms\": %d, \"clock_khz\": %d, \"err\": \"%s\"}\n", S, clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
