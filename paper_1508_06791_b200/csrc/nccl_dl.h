// nccl_dl.h -- NCCL resolved at run time from the libnccl.so.2 already loaded
// in the process (the one torch.distributed uses), so libjacc.so has no link
// dependency on NCCL and uses exactly the communicator's library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace jacc_nccl {
enum { kInt32 = 2, kFloat32 = 7 };   // ncclDataType_t values (nccl.h)
int allreduce_sum(const void *send, void *recv, uint64_t count, int dtype, void *comm, cudaStream_t st);
int allgather(const void *send, void *recv, uint64_t sendcount, int dtype, void *comm, cudaStream_t st);
int broadcast(const void *send, void *recv, uint64_t count, int dtype, int root, void *comm, cudaStream_t st);
int halo_exchange(const float *first, const float *last, float *top, float *bottom, uint64_t count, int rank,
                  int world, void *comm, cudaStream_t st);
const char *last_error();
}  // namespace jacc_nccl
