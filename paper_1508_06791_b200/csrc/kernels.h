// kernels.h -- internal launchers of the sm_100a kernels (not part of the ABI).
// Each launcher validates nothing the runtime already validated, launches on
// `st`, adds the number of CUDA kernels it launched to *launches and returns
// the launch status.  Every kernel is grid-stride or tiled, so the advisory
// schedule (reading R15) never changes a result.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "jacc.h"

namespace jacc_k {

// JACC_GRAPH_P2P (peer.cuh): the windows of all ranks as mapped in this
// process (base[rank] = the local window), and one collective task's slot +
// window offset (allreduce: staging area; allgather / broadcast: receive
// buffer).  Passed to kernels by value.
struct PeerCtx {
    char *base[JACC_PEER_MAX];
    char *self;   // == base[rank]: device code never indexes base[] with a runtime value
    int rank, world;
};
struct PeerOp {
    PeerCtx ctx;
    int slot;
    int64_t off;
};
constexpr size_t kPeerHeaderBytes = 256 * 1024;   // == peer::kHeaderBytes
constexpr int kPeerSlots = 1024;                  // == peer::kSlots

int sm_count();   // SMs of the current device (148 on B200), cached per device
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device);
// thread-safe (graphs of different devices may launch from different threads)
cudaError_t set_max_dyn_smem(const void *kernel, int bytes);
// resident blocks per SM of `kernel` at `block` threads on the current device
int blocks_per_sm(const void *kernel, int block, int dyn_smem);
// cudaOccupancyMaxActiveClusters for a launch config (only its cluster attribute, block and
// dynamic smem matter), cached; 0 when no such cluster can be resident or the query fails
int max_active_clusters(const void *kernel, const cudaLaunchConfig_t *cfg);

// c = a + b
cudaError_t vadd_f32(const float *a, const float *b, float *c, int64_t n,
                     const jacc_schedule_t *s, cudaStream_t st, int *launches);

// out[0] += sum(x) (out pre-zeroed by the runtime for W)
size_t reduce_ws_bytes(int64_t n);
// assign: out[0] = sum (W output, no memset) instead of out[0] += sum
cudaError_t reduce_sum_f32(const float *x, int64_t n, float *out, void *ws,
                           const jacc_schedule_t *s, cudaStream_t st, int *launches, bool assign = false,
                           const PeerOp *allreduce = nullptr);  // fused allreduce(out)
// the runtime's "merge" of vadd -> reduce: c = a + b, out[0] += sum(c)
bool vadd_reduce_fusable(const float *a, const float *b, const float *c);
cudaError_t vadd_reduce_f32(const float *a, const float *b, float *c, int64_t n, float *out, void *ws,
                            const jacc_schedule_t *s_reduce, cudaStream_t st, int *launches, bool assign = false,
                            const PeerOp *allreduce = nullptr);

// bins[k] += #{keys == k}
size_t histogram_ws_bytes(int64_t n, int nbins);
// assign: bins = counts (a W output, instead of a memset + add); else bins += counts
cudaError_t histogram_i32(const int32_t *keys, int64_t n, int32_t *bins, int nbins, void *ws,
                          const jacc_schedule_t *s, cudaStream_t st, int *launches,
                          const PeerOp *allreduce = nullptr,   // fused allreduce(bins), nbins <= 256, n > 0
                          bool assign = false);

// APARAPI Black-Scholes
cudaError_t blackscholes_f32(const float *u, float *call, float *put, int64_t n,
                             const jacc_schedule_t *s, cudaStream_t st, int *launches);
cudaError_t blackscholes_soa_f32(const float *S, const float *K, const float *T, const float *R,
                                 const float *V, float *call, float *put, int64_t n,
                                 const jacc_schedule_t *s, cudaStream_t st, int *launches);

// C = A.B
size_t sgemm_ws_bytes(const jacc_sgemm_params_t *p);
cudaError_t sgemm_f32(const float *A, const float *B, float *C, const jacc_sgemm_params_t *p,
                      void *ws, cudaStream_t st, int *launches);

// north_star N-body step
size_t nbody_ws_bytes(int64_t n_src, int64_t n_tgt);
cudaError_t nbody_step_f32(const float4 *pos_src, int64_t n_src, float4 *vel, float4 *pos_out,
                           int64_t n_tgt, const jacc_nbody_params_t *p, void *ws,
                           const jacc_schedule_t *s, cudaStream_t st, int *launches,
                           const PeerOp *allgather = nullptr);  // fused allgather(pos_out), n_tgt > 0

// JACC_GRAPH_P2P standalone collectives (peer.cu)
size_t peer_allreduce_stage_bytes(int64_t n, int esz, int world);
cudaError_t peer_allreduce(const PeerOp &op, void *buf, int64_t n, bool is_int, cudaStream_t st, int *launches);
cudaError_t peer_allgather(const PeerOp &op, const void *send, int64_t bytes, cudaStream_t st, int *launches);
cudaError_t peer_broadcast(const PeerOp &op, int root, int64_t bytes, cudaStream_t st, int *launches);
// every rank: returns (on the stream) once all ranks reached it -- used before
// a window is unmapped and freed (a peer may still owe it a flag store)
cudaError_t peer_barrier(const PeerCtx &c, int slot, cudaStream_t st);
constexpr int kPeerBarrierSlot = kPeerSlots - 1;   // reserved: collective tasks use 0 .. kPeerSlots - 2

// 2D convolution
cudaError_t conv2d_f32(const float *img, int64_t H_in, int64_t W, const float *filt, int radius, float *out,
                       int64_t y_off, int64_t H, cudaStream_t st, int *launches);
// JACC_OP_HALO_EXCHANGE_F32 (row bands of an image, SPMD): ext = [r rows of
// the band above][band][r rows of the band below], zeros past the image
size_t peer_halo_stage_bytes(int64_t W, int radius);
cudaError_t peer_halo(const PeerOp &op, const float *band, float *ext, int64_t rows, int64_t W, int radius,
                      cudaStream_t st, int *launches);
cudaError_t halo_local(const float *band, float *ext, int64_t rows, int64_t W, int radius, bool top_zero,
                       bool bottom_zero, cudaStream_t st, int *launches);

// correlation matrix
size_t corr_ws_bytes(int64_t ta, int64_t tb, int64_t words);
cudaError_t corr_popc_u32(const uint32_t *A, int64_t ta, const uint32_t *B, int64_t tb, int64_t words, int32_t *C,
                          void *ws, cudaStream_t st, int *launches);

// SpMV CSR
cudaError_t spmv_csr_f32(const int32_t *row_ptr, const int32_t *col, const float *val, const float *x, float *y,
                         int64_t n, int64_t nnz, cudaStream_t st, int *launches);

}  // namespace jacc_k
