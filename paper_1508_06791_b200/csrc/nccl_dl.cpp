// nccl_dl.cpp -- see nccl_dl.h.  nccl.h supplies the types only; no symbol of
// libnccl is linked: the functions are looked up with dlsym at first use.
#include "nccl_dl.h"

#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <string>

namespace jacc_nccl {
namespace {
typedef ncclResult_t (*allreduce_t)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                    cudaStream_t);
typedef ncclResult_t (*allgather_t)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*broadcast_t)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
typedef const char *(*errstr_t)(ncclResult_t);
typedef ncclResult_t (*sendrecv_t)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*send_t)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*group_t)();

struct Api {
    allreduce_t allreduce = nullptr;
    allgather_t allgather = nullptr;
    broadcast_t broadcast = nullptr;
    errstr_t errstr = nullptr;
    send_t send = nullptr;
    sendrecv_t recv = nullptr;
    group_t gstart = nullptr, gend = nullptr;
    bool ok = false;
};
Api g_api;
std::once_flag g_once;
thread_local std::string g_err;

void load() {
    // Prefer the copy already mapped into the process (torch's), then any.
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    g_api.allreduce = (allreduce_t)dlsym(h, "ncclAllReduce");
    g_api.allgather = (allgather_t)dlsym(h, "ncclAllGather");
    g_api.broadcast = (broadcast_t)dlsym(h, "ncclBroadcast");
    g_api.errstr = (errstr_t)dlsym(h, "ncclGetErrorString");
    g_api.send = (send_t)dlsym(h, "ncclSend");
    g_api.recv = (sendrecv_t)dlsym(h, "ncclRecv");
    g_api.gstart = (group_t)dlsym(h, "ncclGroupStart");
    g_api.gend = (group_t)dlsym(h, "ncclGroupEnd");
    g_api.ok = g_api.allreduce && g_api.allgather && g_api.broadcast && g_api.errstr;
}

int check(ncclResult_t r) {
    if (r == ncclSuccess) return 0;
    g_err = g_api.errstr ? g_api.errstr(r) : "nccl error";
    return (int)r;
}

bool ready() {
    std::call_once(g_once, load);
    if (!g_api.ok) g_err = "libnccl.so.2 not found in the process (import torch / init NCCL first)";
    return g_api.ok;
}
}  // namespace

int allreduce_sum(const void *send, void *recv, uint64_t count, int dtype, void *comm, cudaStream_t st) {
    if (!ready()) return -1;
    return check(g_api.allreduce(send, recv, count, (ncclDataType_t)dtype, ncclSum, (ncclComm_t)comm, st));
}
int allgather(const void *send, void *recv, uint64_t sendcount, int dtype, void *comm, cudaStream_t st) {
    if (!ready()) return -1;
    return check(g_api.allgather(send, recv, sendcount, (ncclDataType_t)dtype, (ncclComm_t)comm, st));
}
int broadcast(const void *send, void *recv, uint64_t count, int dtype, int root, void *comm, cudaStream_t st) {
    if (!ready()) return -1;
    return check(g_api.broadcast(send, recv, count, (ncclDataType_t)dtype, root, (ncclComm_t)comm, st));
}
// Halo exchange of row bands (JACC_OP_HALO_EXCHANGE_F32): one NCCL group of
// point-to-point calls -- first `count` floats of band to rank-1's bottom
// halo, last `count` to rank+1's top halo, and the mirror receives.
int halo_exchange(const float *first, const float *last, float *top, float *bottom, uint64_t count, int rank,
                  int world, void *comm, cudaStream_t st) {
    if (!ready()) return -1;
    if (!g_api.send || !g_api.recv || !g_api.gstart || !g_api.gend) {
        g_err = "ncclSend/ncclRecv not found";
        return -1;
    }
    ncclComm_t c = (ncclComm_t)comm;
    int r = check(g_api.gstart());
    if (r) return r;
    if (rank > 0) {
        if ((r = check(g_api.send(first, count, ncclFloat32, rank - 1, c, st)))) return r;
        if ((r = check(g_api.recv(top, count, ncclFloat32, rank - 1, c, st)))) return r;
    }
    if (rank < world - 1) {
        if ((r = check(g_api.send(last, count, ncclFloat32, rank + 1, c, st)))) return r;
        if ((r = check(g_api.recv(bottom, count, ncclFloat32, rank + 1, c, st)))) return r;
    }
    return check(g_api.gend());
}
const char *last_error() { return g_err.c_str(); }
}  // namespace jacc_nccl
