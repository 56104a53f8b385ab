// runtime.cpp -- the Jacc task-graph runtime behind include/jacc.h.
//
// PAPER.md §2 / §2.3 and §3.2.1:
//   task graph (DAG) -> dependency inference -> lowering into
//   transfers / kernels / collectives -> elimination of
//   redundant transfers + out-of-order issue of independent kernels (P:61,
//   P:95) -> traversal-based issue -> sync / commit (P:169-171,
//   P:214), with per-device persistent state (reading R5).
//
// The planner is pure C++ (no CUDA call) so graphs can be built, planned and
// dumped on a machine without a GPU; the issuer uses the CUDA runtime, the
// sm_100a kernels (kernels.h) and NCCL resolved at run time (nccl_dl.cpp).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "jacc.h"
#include "kernels.h"
#include "nccl_dl.h"

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges show in nsys / ncu when a tool is attached

namespace {

thread_local std::string g_last_error;

int fail(int status, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = std::string(jacc_status_string(status)) + ": " + buf;
    return status;
}

size_t dtype_size(int dt) {
    switch (dt) {
        case JACC_F32: return 4;
        case JACC_I32: return 4;
        case JACC_F32X4: return 16;
        default: return 0;
    }
}

const char *op_name(int op) {
    switch (op) {
        case JACC_OP_VADD_F32: return "vadd";
        case JACC_OP_REDUCE_SUM_F32: return "reduce";
        case JACC_OP_HISTOGRAM_I32: return "hist";
        case JACC_OP_BLACKSCHOLES_F32: return "bs";
        case JACC_OP_BLACKSCHOLES_SOA_F32: return "bs_soa";
        case JACC_OP_SGEMM_F32: return "sgemm";
        case JACC_OP_NBODY_STEP_F32: return "nbody";
        case JACC_OP_ALLREDUCE_SUM: return "allreduce";
        case JACC_OP_ALLGATHER: return "allgather";
        case JACC_OP_BROADCAST: return "broadcast";
        case JACC_OP_CONV2D_F32: return "conv2d";
        case JACC_OP_CORR_POPC_U32: return "corr";
        case JACC_OP_SPMV_CSR_F32: return "spmv";
        case JACC_OP_HALO_EXCHANGE_F32: return "halo";
        default: return "?";
    }
}

bool is_collective(int op) {
    return op == JACC_OP_ALLREDUCE_SUM || op == JACC_OP_ALLGATHER || op == JACC_OP_BROADCAST ||
           op == JACC_OP_HALO_EXCHANGE_F32;
}

// index of the @Atomic(op=ADD) output of an op (auto-zeroed in W mode), or -1
int atomic_out(int op) {
    return (op == JACC_OP_REDUCE_SUM_F32 || op == JACC_OP_HISTOGRAM_I32) ? 1 : -1;
}

enum { ST_BUILDING = 0, ST_EXECUTING = 1, ST_DONE = 2, ST_FAILED = 3 };

struct Buffer {
    uintptr_t host = 0;     // host range start (or the device pointer for DEVICE)
    size_t bytes = 0;
    bool device = false;    // JACC_ARG_DEVICE: caller-owned device memory
    bool cachable = false;  // JACC_ARG_CACHABLE on any use
    void *dptr = nullptr;   // graph-owned device copy (or == host for DEVICE)
    bool dev_current = false;  // device copy == host value at the end of the last execute
    bool invalidated = false;
    bool in_window = false; // device copy lives in the P2P window (freed with it)
    cudaEvent_t ev_h2d = nullptr;
};

struct TaskArg {
    int buf;
    uint64_t count;
    int dtype;
    uint32_t access;
    uint32_t flags;
};

struct Task {
    int op;
    std::vector<TaskArg> args;
    std::vector<unsigned char> params;
    jacc_schedule_t sched;
    bool has_sched = false;
    std::vector<int> preds;   // inferred edges p -> this
    int stream = 0;           // planned stream index (-1 = comm stream)
    void *ws = nullptr;
    size_t ws_bytes = 0;
    cudaEvent_t ev_start = nullptr, ev_end = nullptr;   // timing
    cudaEvent_t ev_dep = nullptr;                       // dependency (no timing)
    float ms = 0.f;
    int slot = -1;              // JACC_GRAPH_P2P: collective slot (peer.cuh)
    int fused_into = -1;        // issue: task whose kernel also runs this one (merge), else -1
    int64_t peer_off = -1;      // JACC_GRAPH_P2P allreduce: staging offset in the window
};

enum ActKind { A_H2D, A_MEMSET0, A_KERNEL, A_COLLECTIVE, A_D2H };
struct Action {
    ActKind kind;
    int buf;    // H2D / MEMSET0 / D2H
    int task;   // KERNEL / COLLECTIVE / MEMSET0 (owner task)
};

}  // namespace

struct jacc_graph {
    jacc_config_t cfg;
    int state = ST_BUILDING;
    std::vector<Buffer> bufs;
    std::vector<Task> tasks;
    std::vector<Action> plan;
    std::vector<int> last_writer;
    bool planned = false;
    std::vector<char> plan_dev_valid;   // residency the plan was made for (re-plan when it changes)
    std::vector<std::vector<int>> memset_bufs;   // per task: its MEMSET0 buffers (from the plan)
    std::vector<int> h2d_order;         // plan indices of the H2D actions, critical path first
    bool have_times = false;
    // resources
    bool res_ready = false;
    int n_streams = 0;
    cudaStream_t compute[JACC_MAX_STREAMS] = {};
    bool own_compute = false;
    cudaStream_t h2d = nullptr, d2h = nullptr, comm = nullptr;
    bool own_h2d = false, own_d2h = false, own_comm = false;
    jacc_stats_t stats;
    int pending_error = JACC_OK;
    // JACC_GRAPH_REPLAY: captured CUDA graph of the issued action list
    cudaGraphExec_t exec = nullptr;
    std::vector<Action> exec_plan;   // the plan `exec` was captured from
    uint64_t exec_launches = 0;
    bool exec_failed = false;        // capture impossible for this plan: issue directly
    cudaEvent_t ev_fork = nullptr;
    std::vector<cudaEvent_t> ev_join;
    bool capturing = false;          // issue() runs under stream capture
    bool last_was_replay = false;    // current execute = one graph launch on compute[0]
    // JACC_GRAPH_P2P: symmetric window (peer.cuh) and the peers' mappings
    char *win = nullptr;
    size_t win_bytes = 0, win_top = 0;   // bump allocator (same sequence on every rank)
    char *peer_base[JACC_PEER_MAX] = {};
    bool peer_connected = false;
};

// ---------------------------------------------------------------- helpers
namespace {

int n_streams_of(const jacc_graph *g) {
    if (g->cfg.flags & (JACC_GRAPH_NAIVE | JACC_GRAPH_SERIAL)) return 1;
    return g->cfg.n_compute > 0 ? g->cfg.n_compute : 4;
}

bool p2p(const jacc_graph *g) { return g->cfg.flags & JACC_GRAPH_P2P; }

// Bump-allocate from the P2P window (256-byte aligned); -1 when full.
int64_t win_alloc(jacc_graph *g, size_t bytes) {
    const size_t off = (g->win_top + 255) & ~(size_t)255;
    if (!g->win || off + bytes > g->win_bytes) return -1;
    g->win_top = off + (bytes ? bytes : 16);
    return (int64_t)off;
}

// Offset of [p, p + bytes) inside the local window, or -1.
int64_t win_off(const jacc_graph *g, const void *p, size_t bytes) {
    const char *c = (const char *)p;
    if (!g->win || c < g->win + jacc_k::kPeerHeaderBytes || c + bytes > g->win + g->win_bytes) return -1;
    return (int64_t)(c - g->win);
}

jacc_k::PeerCtx peer_ctx(const jacc_graph *g) {
    jacc_k::PeerCtx c{};
    for (int q = 0; q < g->cfg.world; ++q) c.base[q] = q == g->cfg.rank ? g->win : g->peer_base[q];
    c.self = g->win;
    c.rank = g->cfg.rank;
    c.world = g->cfg.world;
    return c;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(JACC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(call)                                                   \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);        \
    } while (0)

void *dev_alloc(jacc_graph *g, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (g->cfg.alloc) return g->cfg.alloc(bytes, g->cfg.device, (void *)g->compute[0], g->cfg.alloc_ctx);
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    return p;
}

void dev_free(jacc_graph *g, void *p, size_t bytes) {
    if (!p) return;
    if (g->cfg.free) g->cfg.free(p, bytes, g->cfg.device, (void *)g->compute[0], g->cfg.alloc_ctx);
    else cudaFree(p);
}

// Validate an op's signature: arg count, access, dtype, counts, params (SURVEY §8b "Ops").
int validate(const jacc_graph *g, int op, const jacc_arg_t *a, int n, const void *params,
             size_t psz) {
    auto need = [&](int k) -> int {
        if (n != k) return fail(JACC_ERR_INVALID_ARG, "%s takes %d args, got %d", op_name(op), k, n);
        return JACC_OK;
    };
    auto acc = [&](int i, uint32_t allowed_mask) -> int {
        // allowed_mask: bit (1 << access); access is READ, WRITE or READWRITE
        if (a[i].access < JACC_READ || a[i].access > JACC_READWRITE || !((1u << a[i].access) & allowed_mask))
            return fail(JACC_ERR_ACCESS, "%s arg %d: access %u not allowed", op_name(op), i, a[i].access);
        return JACC_OK;
    };
    auto dt = [&](int i, int d) -> int {
        if (a[i].dtype != d) return fail(JACC_ERR_INVALID_ARG, "%s arg %d: dtype %d, want %d", op_name(op), i, a[i].dtype, d);
        return JACC_OK;
    };
    const uint32_t R = 1u << JACC_READ, W = 1u << JACC_WRITE, RW = 1u << JACC_READWRITE;
    int s;
#define T(x) if ((s = (x)) != JACC_OK) return s
    switch (op) {
        case JACC_OP_VADD_F32:
            T(need(3)); T(acc(0, R)); T(acc(1, R)); T(acc(2, W));
            for (int i = 0; i < 3; ++i) T(dt(i, JACC_F32));
            if (a[1].count != a[0].count || a[2].count != a[0].count)
                return fail(JACC_ERR_INVALID_ARG, "vadd: counts differ");
            break;
        case JACC_OP_REDUCE_SUM_F32:
            T(need(2)); T(acc(0, R)); T(acc(1, W | RW)); T(dt(0, JACC_F32)); T(dt(1, JACC_F32));
            if (a[1].count != 1) return fail(JACC_ERR_INVALID_ARG, "reduce: out must have count 1");
            break;
        case JACC_OP_HISTOGRAM_I32: {
            T(need(2)); T(acc(0, R)); T(acc(1, W | RW)); T(dt(0, JACC_I32)); T(dt(1, JACC_I32));
            if (!params || psz < sizeof(jacc_hist_params_t)) return fail(JACC_ERR_INVALID_ARG, "hist: params");
            int nb = ((const jacc_hist_params_t *)params)->nbins;
            if (nb < 1 || nb > 4096) return fail(JACC_ERR_UNSUPPORTED, "hist: nbins %d not in [1, 4096]", nb);
            if ((int64_t)a[1].count != nb) return fail(JACC_ERR_INVALID_ARG, "hist: bins count != nbins");
            break;
        }
        case JACC_OP_BLACKSCHOLES_F32:
            T(need(3)); T(acc(0, R)); T(acc(1, W)); T(acc(2, W));
            for (int i = 0; i < 3; ++i) T(dt(i, JACC_F32));
            if (a[1].count != a[0].count || a[2].count != a[0].count)
                return fail(JACC_ERR_INVALID_ARG, "bs: counts differ");
            break;
        case JACC_OP_BLACKSCHOLES_SOA_F32:
            T(need(7));
            for (int i = 0; i < 5; ++i) T(acc(i, R));
            T(acc(5, W)); T(acc(6, W));
            for (int i = 0; i < 7; ++i) {
                T(dt(i, JACC_F32));
                if (a[i].count != a[0].count) return fail(JACC_ERR_INVALID_ARG, "bs_soa: counts differ");
            }
            break;
        case JACC_OP_SGEMM_F32: {
            T(need(3)); T(acc(0, R)); T(acc(1, R)); T(acc(2, W));
            for (int i = 0; i < 3; ++i) T(dt(i, JACC_F32));
            if (!params || psz < sizeof(jacc_sgemm_params_t)) return fail(JACC_ERR_INVALID_ARG, "sgemm: params");
            const jacc_sgemm_params_t *p = (const jacc_sgemm_params_t *)params;
            if (p->M < 0 || p->N < 0 || p->K < 0 || p->lda < p->K || p->ldb < p->N || p->ldc < p->N)
                return fail(JACC_ERR_INVALID_ARG, "sgemm: bad shape/strides");
            if (p->mode != JACC_SGEMM_3XTF32 && p->mode != JACC_SGEMM_FFMA)
                return fail(JACC_ERR_INVALID_ARG, "sgemm: mode %d", p->mode);
            auto span = [](int64_t rows, int64_t ld, int64_t cols) -> uint64_t {
                return rows == 0 || cols == 0 ? 0 : (uint64_t)((rows - 1) * ld + cols);
            };
            if (a[0].count < span(p->M, p->lda, p->K) || a[1].count < span(p->K, p->ldb, p->N) ||
                a[2].count < span(p->M, p->ldc, p->N))
                return fail(JACC_ERR_INVALID_ARG, "sgemm: buffer smaller than the shape");
            break;
        }
        case JACC_OP_NBODY_STEP_F32: {
            T(need(3)); T(acc(0, R)); T(acc(1, RW)); T(acc(2, W));
            for (int i = 0; i < 3; ++i) T(dt(i, JACC_F32X4));
            if (!params || psz < sizeof(jacc_nbody_params_t)) return fail(JACC_ERR_INVALID_ARG, "nbody: params");
            const jacc_nbody_params_t *p = (const jacc_nbody_params_t *)params;
            if (a[2].count != a[1].count) return fail(JACC_ERR_INVALID_ARG, "nbody: vel/pos_out counts differ");
            if (p->tgt_offset < 0 || (uint64_t)p->tgt_offset + a[1].count > a[0].count)
                return fail(JACC_ERR_INVALID_ARG, "nbody: targets outside pos_src");
            if (!(p->eps2 > 0.f)) return fail(JACC_ERR_INVALID_ARG, "nbody: eps2 must be > 0");
            if (a[0].count > (uint64_t)65535 * 2048)
                return fail(JACC_ERR_UNSUPPORTED, "nbody: %llu sources > 65535 chunks of 2048",
                            (unsigned long long)a[0].count);
            break;
        }
        case JACC_OP_ALLREDUCE_SUM:
            T(need(1)); T(acc(0, RW));
            if (a[0].dtype != JACC_F32 && a[0].dtype != JACC_I32)
                return fail(JACC_ERR_INVALID_ARG, "allreduce: dtype must be f32 or i32");
            break;
        case JACC_OP_ALLGATHER:
            T(need(2)); T(acc(0, R)); T(acc(1, W));
            if (a[1].dtype != a[0].dtype) return fail(JACC_ERR_INVALID_ARG, "allgather: dtypes differ");
            if (a[1].count != a[0].count * (uint64_t)g->cfg.world)
                return fail(JACC_ERR_INVALID_ARG, "allgather: recv count != send count * world");
            break;
        case JACC_OP_HALO_EXCHANGE_F32: {
            T(need(2)); T(acc(0, R)); T(acc(1, W)); T(dt(0, JACC_F32)); T(dt(1, JACC_F32));
            if (!params || psz < sizeof(jacc_halo_params_t)) return fail(JACC_ERR_INVALID_ARG, "halo: params");
            const jacc_halo_params_t *p = (const jacc_halo_params_t *)params;
            if (p->radius < 1 || p->rows < 0 || p->W < 0 || a[0].count != (uint64_t)p->rows * (uint64_t)p->W ||
                a[1].count != (uint64_t)(p->rows + 2 * p->radius) * (uint64_t)p->W)
                return fail(JACC_ERR_INVALID_ARG, "halo: counts do not match rows, W, radius");
            if (p->rows < p->radius && g->cfg.world > 1)
                return fail(JACC_ERR_UNSUPPORTED, "halo: band of %lld rows < radius %d",
                            (long long)p->rows, p->radius);
            break;
        }
        case JACC_OP_BROADCAST: {
            T(need(1)); T(acc(0, RW));
            if (!params || psz < sizeof(jacc_bcast_params_t)) return fail(JACC_ERR_INVALID_ARG, "broadcast: params");
            int root = ((const jacc_bcast_params_t *)params)->root;
            if (root < 0 || root >= g->cfg.world) return fail(JACC_ERR_INVALID_ARG, "broadcast: root");
            break;
        }
        case JACC_OP_CONV2D_F32: {
            T(need(3)); T(acc(0, R)); T(acc(1, R)); T(acc(2, W));
            for (int i = 0; i < 3; ++i) T(dt(i, JACC_F32));
            if (!params || psz < sizeof(jacc_conv2d_params_t)) return fail(JACC_ERR_INVALID_ARG, "conv2d: params");
            const jacc_conv2d_params_t *p = (const jacc_conv2d_params_t *)params;
            if (p->radius < 1 || p->radius > 4) return fail(JACC_ERR_UNSUPPORTED, "conv2d: radius %d", p->radius);
            const uint64_t k = 2 * p->radius + 1;
            if (p->flags & ~JACC_CONV2D_HALO_ROWS) return fail(JACC_ERR_INVALID_ARG, "conv2d: unknown flags");
            const uint64_t h_in = (uint64_t)p->H + ((p->flags & JACC_CONV2D_HALO_ROWS) ? 2 * p->radius : 0);
            if (p->H < 0 || p->W < 0 || a[0].count != h_in * (uint64_t)p->W ||
                a[2].count != (uint64_t)p->H * (uint64_t)p->W || a[1].count != k * k)
                return fail(JACC_ERR_INVALID_ARG, "conv2d: counts do not match H x W / filter size");
            break;
        }
        case JACC_OP_CORR_POPC_U32: {
            T(need(3)); T(acc(0, R)); T(acc(1, R)); T(acc(2, W));
            for (int i = 0; i < 3; ++i) T(dt(i, JACC_I32));
            if (!params || psz < sizeof(jacc_corr_params_t)) return fail(JACC_ERR_INVALID_ARG, "corr: params");
            const jacc_corr_params_t *p = (const jacc_corr_params_t *)params;
            if (p->ta < 0 || p->tb < 0 || p->words < 0 || a[0].count != (uint64_t)p->ta * (uint64_t)p->words ||
                a[1].count != (uint64_t)p->tb * (uint64_t)p->words || a[2].count != (uint64_t)p->ta * (uint64_t)p->tb)
                return fail(JACC_ERR_INVALID_ARG, "corr: counts do not match ta, tb, words");
            break;
        }
        case JACC_OP_SPMV_CSR_F32: {
            T(need(5));
            for (int i = 0; i < 4; ++i) T(acc(i, R));
            T(acc(4, W)); T(dt(0, JACC_I32)); T(dt(1, JACC_I32)); T(dt(2, JACC_F32)); T(dt(3, JACC_F32));
            T(dt(4, JACC_F32));
            if (!params || psz < sizeof(jacc_spmv_params_t)) return fail(JACC_ERR_INVALID_ARG, "spmv: params");
            const jacc_spmv_params_t *p = (const jacc_spmv_params_t *)params;
            if (p->n < 0 || a[0].count != (uint64_t)p->n + 1 || a[1].count != a[2].count ||
                a[3].count != (uint64_t)p->ncols || a[4].count != (uint64_t)p->n)
                return fail(JACC_ERR_INVALID_ARG, "spmv: counts do not match n, ncols, nnz");
            break;
        }
        default:
            return fail(JACC_ERR_INVALID_ARG, "unknown op %d", op);
    }
#undef T
    for (int i = 0; i < n; ++i) {
        if (!a[i].ptr && a[i].count) return fail(JACC_ERR_INVALID_ARG, "arg %d: NULL pointer", i);
        if (dtype_size(a[i].dtype) == 0) return fail(JACC_ERR_INVALID_ARG, "arg %d: dtype", i);
        if (a[i].flags & ~(JACC_ARG_DEVICE | JACC_ARG_CACHABLE))
            return fail(JACC_ERR_INVALID_ARG, "arg %d: unknown flags", i);
    }
    return JACC_OK;
}

// Find or register the buffer of an argument by its exact byte range.
int resolve_buffer(jacc_graph *g, const jacc_arg_t &a, std::vector<Buffer> &newbufs, int *id) {
    uintptr_t lo = (uintptr_t)a.ptr;
    size_t bytes = a.count * dtype_size(a.dtype);
    bool dev = a.flags & JACC_ARG_DEVICE;
    auto check = [&](const Buffer &b, int idx) -> int {
        if (b.host == lo && b.bytes == bytes) {
            if (b.device != dev) return fail(JACC_ERR_ALIAS, "buffer %p used both as DEVICE and host", a.ptr);
            *id = idx;
            return 1;
        }
        if (bytes && b.bytes && lo < b.host + b.bytes && b.host < lo + bytes)
            return fail(JACC_ERR_ALIAS, "range [%p, +%zu) partially overlaps buffer %d", a.ptr, bytes, idx);
        return 0;
    };
    int nb = (int)g->bufs.size();
    for (int i = 0; i < nb; ++i) {
        int r = check(g->bufs[i], i);
        if (r == 1) return JACC_OK;
        if (r != 0) return r;
    }
    for (int i = 0; i < (int)newbufs.size(); ++i) {
        int r = check(newbufs[i], nb + i);
        if (r == 1) return JACC_OK;
        if (r != 0) return r;
    }
    Buffer b;
    b.host = lo;
    b.bytes = bytes;
    b.device = dev;
    if (dev) b.dptr = a.ptr;
    newbufs.push_back(b);
    *id = nb + (int)newbufs.size() - 1;
    return JACC_OK;
}

// Rough device-time estimate of a task (s) from its algorithmic bytes/flops
// at B200-class rates: only used to ORDER the host->device copies.
double est_cost(const jacc_graph *g, const Task &T) {
    const TaskArg *a = T.args.data();
    const double hbm = 6e12, alu = 5e13, tc = 2.5e14, link = 5e10;
    switch (T.op) {
        case JACC_OP_VADD_F32: return 12.0 * a[0].count / hbm;
        case JACC_OP_REDUCE_SUM_F32:
        case JACC_OP_HISTOGRAM_I32: return 4.0 * a[0].count / hbm;
        case JACC_OP_BLACKSCHOLES_F32: return 12.0 * a[0].count / hbm;
        case JACC_OP_BLACKSCHOLES_SOA_F32: return 28.0 * a[0].count / hbm;
        case JACC_OP_SGEMM_F32: {
            const jacc_sgemm_params_t *p = (const jacc_sgemm_params_t *)T.params.data();
            return 2.0 * p->M * p->N * p->K / tc;
        }
        case JACC_OP_NBODY_STEP_F32: return 20.0 * a[0].count * a[1].count / alu;
        case JACC_OP_CONV2D_F32: return 8.0 * a[0].count / hbm;
        case JACC_OP_HALO_EXCHANGE_F32: return 8.0 * a[0].count / hbm;
        case JACC_OP_CORR_POPC_U32: {
            const jacc_corr_params_t *p = (const jacc_corr_params_t *)T.params.data();
            return 3.0 * p->ta * p->tb * p->words / alu;
        }
        case JACC_OP_SPMV_CSR_F32: return 12.0 * a[1].count / hbm;
        default: return (double)a[0].count * dtype_size(a[0].dtype) / link;
    }
}

// "Nodes' re-organization ... early kernel scheduling" (reading R6):
// host->device copies are issued in order of the critical path (estimated
// device time from the consuming task to the end of the graph), so the
// longest chain's inputs land first and its kernels start while the other
// inputs are still crossing PCIe.  The lowered action list itself (and so
// every counted copy) is unchanged.
// Bottom level of every task: its estimated cost plus the longest estimated
// path through its successors to the end of the graph.
std::vector<double> bottom_level(const jacc_graph *g) {
    const int nt = (int)g->tasks.size();
    std::vector<double> prio(nt, 0.0);
    std::vector<std::vector<int>> succ(nt);
    for (int t = 0; t < nt; ++t)
        for (int p : g->tasks[t].preds) succ[p].push_back(t);
    for (int t = nt - 1; t >= 0; --t) {
        double m = 0.0;
        for (int s : succ[t]) m = std::max(m, prio[s]);
        prio[t] = est_cost(g, g->tasks[t]) + m;
    }
    return prio;
}

std::vector<int> h2d_issue_order(const jacc_graph *g) {
    const std::vector<double> prio = bottom_level(g);
    std::vector<int> idx;
    for (int i = 0; i < (int)g->plan.size(); ++i)
        if (g->plan[i].kind == A_H2D) idx.push_back(i);
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int x, int y) { return prio[g->plan[x].task] > prio[g->plan[y].task]; });
    return idx;
}

// ------------------------------------------------------------- planner
// Transfer model G.3 (reading R3) -- identical to the
// oracle's oracle/graph_model.py:plan, which tests/ compare against.
std::vector<char> initial_dev_valid(const jacc_graph *g) {
    std::vector<char> v(g->bufs.size());
    for (size_t b = 0; b < g->bufs.size(); ++b) {
        const Buffer &B = g->bufs[b];
        v[b] = (B.cachable && B.dev_current && !B.invalidated && B.dptr) ? 1 : 0;
    }
    return v;
}

void make_plan(jacc_graph *g) {
    const bool naive = g->cfg.flags & JACC_GRAPH_NAIVE;
    const int nb = (int)g->bufs.size();
    std::vector<char> dev_valid = initial_dev_valid(g), host_valid(nb, 1);
    g->plan_dev_valid = dev_valid;
    g->last_writer.assign(nb, -1);
    g->plan.clear();
    // streams (out-of-order issue, R6): a task with predecessors stays on the
    // stream of its latest one (a chain needs no cross-stream waits); a root
    // task gets a stream by the rank of its critical path among the roots --
    // the longest chains own a stream each, the shortest share the last one
    // -- so a long chain never queues behind a short one whose inputs are
    // copied in late (H2D is issued critical-path first).
    const int ns = n_streams_of(g);
    std::vector<int> root_stream(g->tasks.size(), 0);
    {
        const std::vector<double> prio = bottom_level(g);
        std::vector<int> roots;
        for (int t = 0; t < (int)g->tasks.size(); ++t) {   // chain heads: no kernel predecessor
            if (is_collective(g->tasks[t].op)) continue;
            bool head = true;
            for (int p : g->tasks[t].preds) head = head && is_collective(g->tasks[p].op);
            if (head) roots.push_back(t);
        }
        std::stable_sort(roots.begin(), roots.end(), [&](int x, int y) { return prio[x] > prio[y]; });
        for (int r = 0; r < (int)roots.size(); ++r) root_stream[roots[r]] = std::min(r, ns - 1);
    }
    int next_slot = 0;   // JACC_GRAPH_P2P: collective tasks numbered in insertion order
    for (int t = 0; t < (int)g->tasks.size(); ++t) {
        Task &T = g->tasks[t];
        T.slot = is_collective(T.op) ? next_slot++ : -1;
        if (naive || (g->cfg.flags & JACC_GRAPH_SERIAL)) {
            T.stream = 0;
        } else if (is_collective(T.op)) {
            T.stream = -1;
        } else {
            int s = -2;
            for (int p = (int)T.preds.size() - 1; p >= 0; --p) {
                int ps = g->tasks[T.preds[p]].stream;
                if (ps >= 0) { s = ps; break; }
            }
            if (s < 0) s = root_stream[t];
            T.stream = s;
        }
        const int at = atomic_out(T.op);
        for (const TaskArg &a : T.args) {
            if (g->bufs[a.buf].device) continue;
            if ((a.access & JACC_READ) && (naive || !dev_valid[a.buf])) {
                g->plan.push_back({A_H2D, a.buf, t});
                dev_valid[a.buf] = 1;
            }
        }
        for (int k = 0; k < (int)T.args.size(); ++k)
            if (k == at && T.args[k].access == JACC_WRITE) g->plan.push_back({A_MEMSET0, T.args[k].buf, t});
        g->plan.push_back({is_collective(T.op) ? A_COLLECTIVE : A_KERNEL, -1, t});
        for (const TaskArg &a : T.args) {
            if (a.access & JACC_WRITE) {
                dev_valid[a.buf] = 1;
                host_valid[a.buf] = 0;
                g->last_writer[a.buf] = t;
                if (naive && !g->bufs[a.buf].device) {
                    g->plan.push_back({A_D2H, a.buf, t});
                    host_valid[a.buf] = 1;
                }
            }
        }
    }
    if (!naive) {
        std::vector<int> stale;
        for (int b = 0; b < nb; ++b)
            if (!host_valid[b] && !g->bufs[b].device) stale.push_back(b);
        std::stable_sort(stale.begin(), stale.end(), [&](int x, int y) {
            return g->last_writer[x] < g->last_writer[y];
        });
        for (int b : stale) g->plan.push_back({A_D2H, b, g->last_writer[b]});
    }
    g->memset_bufs.assign(g->tasks.size(), {});
    for (const Action &A : g->plan)
        if (A.kind == A_MEMSET0) g->memset_bufs[A.task].push_back(A.buf);
    g->h2d_order = h2d_issue_order(g);
    g->planned = true;
}

// Re-plan only when a task was added or the residency the plan assumed changed.
void ensure_plan(jacc_graph *g) {
    if (!g->planned || g->plan_dev_valid != initial_dev_valid(g)) make_plan(g);
}

void plan_counts(const jacc_graph *g, jacc_stats_t *s) {
    s->h2d_count = s->h2d_bytes = s->d2h_count = s->d2h_bytes = 0;
    s->memsets = s->kernels = s->collectives = 0;
    for (const Action &a : g->plan) {
        switch (a.kind) {
            case A_H2D: s->h2d_count++; s->h2d_bytes += g->bufs[a.buf].bytes; break;
            case A_D2H: s->d2h_count++; s->d2h_bytes += g->bufs[a.buf].bytes; break;
            case A_MEMSET0: s->memsets++; break;
            case A_KERNEL: s->kernels++; break;
            case A_COLLECTIVE: s->collectives++; break;
        }
    }
}

int merge_partner(const jacc_graph *g, int i);

std::string dump_text(const jacc_graph *g) {
    std::string out;
    char line[256];
    snprintf(line, sizeof line, "graph tasks=%zu buffers=%zu naive=%d\n", g->tasks.size(), g->bufs.size(),
             (g->cfg.flags & JACC_GRAPH_NAIVE) ? 1 : 0);
    out += line;
    for (size_t t = 0; t < g->tasks.size(); ++t) {
        const Task &T = g->tasks[t];
        snprintf(line, sizeof line, "task %zu %s stream=%d args=", t, op_name(T.op), T.stream);
        out += line;
        for (size_t k = 0; k < T.args.size(); ++k) {
            const TaskArg &a = T.args[k];
            const char *m = a.access == JACC_READ ? "R" : a.access == JACC_WRITE ? "W" : "RW";
            snprintf(line, sizeof line, "%sb%d:%s%s", k ? "," : "", a.buf, m,
                     g->bufs[a.buf].device ? ":dev" : "");
            out += line;
        }
        out += "\n";
    }
    for (size_t t = 0; t < g->tasks.size(); ++t)
        for (int p : g->tasks[t].preds) {
            snprintf(line, sizeof line, "edge %d %zu\n", p, t);
            out += line;
        }
    for (const Action &a : g->plan) {
        switch (a.kind) {
            case A_H2D: snprintf(line, sizeof line, "action H2D b%d %zu\n", a.buf, g->bufs[a.buf].bytes); break;
            case A_D2H: snprintf(line, sizeof line, "action D2H b%d %zu\n", a.buf, g->bufs[a.buf].bytes); break;
            case A_MEMSET0: snprintf(line, sizeof line, "action MEMSET0 b%d\n", a.buf); break;
            case A_KERNEL: snprintf(line, sizeof line, "action KERNEL t%d %s\n", a.task, op_name(g->tasks[a.task].op)); break;
            case A_COLLECTIVE: snprintf(line, sizeof line, "action COLLECTIVE t%d %s\n", a.task, op_name(g->tasks[a.task].op)); break;
        }
        out += line;
    }
    if (p2p(g))   // JACC_GRAPH_P2P: collectives fused into their producer's kernel
        for (size_t t = 0; t < g->tasks.size(); ++t) {
            const int j = merge_partner(g, (int)t);
            if (j >= 0 && is_collective(g->tasks[j].op)) {
                snprintf(line, sizeof line, "fuse t%zu %s + t%d %s slot=%d\n", t, op_name(g->tasks[t].op), j,
                         op_name(g->tasks[j].op), g->tasks[j].slot);
                out += line;
            }
        }
    return out;
}

// ------------------------------------------------------------- resources
int ensure_resources(jacc_graph *g) {
    if (g->res_ready) return JACC_OK;
    CK(cudaSetDevice(g->cfg.device));
    g->n_streams = n_streams_of(g);
    if (g->cfg.n_compute > 0) {
        for (int i = 0; i < g->cfg.n_compute; ++i) g->compute[i] = (cudaStream_t)g->cfg.compute[i];
        if (g->n_streams > g->cfg.n_compute) g->n_streams = g->cfg.n_compute;
    } else {
        for (int i = 0; i < g->n_streams; ++i) CK(cudaStreamCreateWithFlags(&g->compute[i], cudaStreamNonBlocking));
        g->own_compute = true;
    }
    const bool naive = g->cfg.flags & JACC_GRAPH_NAIVE;
    if (naive) {
        g->h2d = g->d2h = g->comm = g->compute[0];
    } else {
        if (g->cfg.h2d) g->h2d = (cudaStream_t)g->cfg.h2d;
        else { CK(cudaStreamCreateWithFlags(&g->h2d, cudaStreamNonBlocking)); g->own_h2d = true; }
        if (g->cfg.d2h) g->d2h = (cudaStream_t)g->cfg.d2h;
        else { CK(cudaStreamCreateWithFlags(&g->d2h, cudaStreamNonBlocking)); g->own_d2h = true; }
        if (g->cfg.comm) g->comm = (cudaStream_t)g->cfg.comm;
        else { CK(cudaStreamCreateWithFlags(&g->comm, cudaStreamNonBlocking)); g->own_comm = true; }
    }
    g->res_ready = true;
    return JACC_OK;
}

// The stream a task's work is issued on (a merged task: its host kernel's).
cudaStream_t stream_of(jacc_graph *g, const Task &T) {
    if (T.fused_into >= 0) return stream_of(g, g->tasks[T.fused_into]);
    if (T.stream < 0) return g->comm;
    return g->compute[T.stream % g->n_streams];
}

int peer_init_window(jacc_graph *g, size_t bytes);

// JACC_GRAPH_P2P: give every collective task its window memory, before the
// other device copies are allocated.  Allreduce: a staging area (2 epochs x
// world rows).  Allgather / broadcast: the buffer the peers store into must
// sit in the window at the same offset on every rank -- a graph-owned device
// copy is allocated there, a DEVICE argument must come from jacc_peer_alloc.
// Window offsets are handed out in task order, identical on every rank.
int prepare_peer(jacc_graph *g) {
    if (!g->win) {
        if (g->cfg.world > 1) return fail(JACC_ERR_STATE, "P2P graph with world %d: jacc_peer_init/connect first",
                                          g->cfg.world);
        int rc = peer_init_window(g, 0);   // world 1: a local window
        if (rc != JACC_OK) return rc;
    }
    if (g->cfg.world > 1 && !g->peer_connected) return fail(JACC_ERR_STATE, "P2P graph not connected");
    for (Task &T : g->tasks) {
        if (!is_collective(T.op)) continue;
        if (T.slot >= jacc_k::kPeerBarrierSlot)
            return fail(JACC_ERR_UNSUPPORTED, "P2P graph with more than %d collective tasks",
                        jacc_k::kPeerBarrierSlot);
        const TaskArg &a = T.args[0];
        if (T.op == JACC_OP_ALLREDUCE_SUM) {
            if (T.peer_off < 0) {
                T.peer_off = win_alloc(g, jacc_k::peer_allreduce_stage_bytes((int64_t)a.count, 4, g->cfg.world));
                if (T.peer_off < 0) return fail(JACC_ERR_OOM, "P2P window full (allreduce staging)");
            }
            continue;
        }
        if (T.op == JACC_OP_HALO_EXCHANGE_F32) {   // staging for the neighbours' edge rows
            if (T.peer_off < 0) {
                const jacc_halo_params_t *hp = (const jacc_halo_params_t *)T.params.data();
                T.peer_off = win_alloc(g, jacc_k::peer_halo_stage_bytes(hp->W, hp->radius));
                if (T.peer_off < 0) return fail(JACC_ERR_OOM, "P2P window full (halo staging)");
            }
            continue;
        }
        Buffer &B = g->bufs[T.args[T.op == JACC_OP_ALLGATHER ? 1 : 0].buf];
        if (B.device) {
            if (win_off(g, B.dptr, B.bytes) < 0)
                return fail(JACC_ERR_INVALID_ARG, "%s: DEVICE buffer %p is not in the P2P window (jacc_peer_alloc)",
                            op_name(T.op), B.dptr);
        } else if (!B.in_window) {
            if (B.dptr) dev_free(g, B.dptr, B.bytes);   // allocated before it became a P2P receiver
            const int64_t off = win_alloc(g, B.bytes);
            if (off < 0) return fail(JACC_ERR_OOM, "P2P window full (%zu-byte buffer)", B.bytes);
            B.dptr = g->win + off;
            B.in_window = true;
            B.dev_current = false;
        }
    }
    return JACC_OK;
}

int prepare_memory(jacc_graph *g) {
    if (p2p(g)) {
        int rc = prepare_peer(g);
        if (rc != JACC_OK) return rc;
    }
    for (Buffer &B : g->bufs) {
        if (!B.device && !B.dptr) {
            B.dptr = dev_alloc(g, B.bytes);
            if (!B.dptr) return fail(JACC_ERR_OOM, "device copy of %zu bytes", B.bytes);
            B.dev_current = false;
        }
        if (!B.ev_h2d) CK(cudaEventCreateWithFlags(&B.ev_h2d, cudaEventDisableTiming));
    }
    for (Task &T : g->tasks) {
        if (!(g->cfg.flags & JACC_GRAPH_NO_TIMING)) {
            if (!T.ev_start) CK(cudaEventCreate(&T.ev_start));
            if (!T.ev_end) CK(cudaEventCreate(&T.ev_end));
        }
        if (!T.ev_dep) CK(cudaEventCreateWithFlags(&T.ev_dep, cudaEventDisableTiming));
        size_t need = 0;
        const TaskArg *a = T.args.data();
        switch (T.op) {
            case JACC_OP_REDUCE_SUM_F32: need = jacc_k::reduce_ws_bytes((int64_t)a[0].count); break;
            case JACC_OP_HISTOGRAM_I32:
                need = jacc_k::histogram_ws_bytes((int64_t)a[0].count,
                                                  ((const jacc_hist_params_t *)T.params.data())->nbins);
                break;
            case JACC_OP_SGEMM_F32: need = jacc_k::sgemm_ws_bytes((const jacc_sgemm_params_t *)T.params.data()); break;
            case JACC_OP_NBODY_STEP_F32: need = jacc_k::nbody_ws_bytes((int64_t)a[0].count, (int64_t)a[1].count); break;
            case JACC_OP_CORR_POPC_U32: {
                const jacc_corr_params_t *cp = (const jacc_corr_params_t *)T.params.data();
                need = jacc_k::corr_ws_bytes(cp->ta, cp->tb, cp->words);
                break;
            }
            default: break;
        }
        if (need > T.ws_bytes) {
            dev_free(g, T.ws, T.ws_bytes);
            T.ws = dev_alloc(g, need);
            if (!T.ws) return fail(JACC_ERR_OOM, "workspace of %zu bytes", need);
            T.ws_bytes = need;
            // workspaces hold self-resetting counters: start zeroed
            CK(cudaMemsetAsync(T.ws, 0, need, g->compute[0]));
            CK(cudaStreamSynchronize(g->compute[0]));
        }
    }
    return JACC_OK;
}

int nccl_dtype(int dt, uint64_t count, uint64_t *n_out) {
    if (dt == JACC_F32X4) { *n_out = count * 4; return jacc_nccl::kFloat32; }
    *n_out = count;
    return dt == JACC_I32 ? jacc_nccl::kInt32 : jacc_nccl::kFloat32;
}

jacc_k::PeerOp peer_op(const jacc_graph *g, const Task &C) {
    jacc_k::PeerOp op{};
    op.ctx = peer_ctx(g);
    op.slot = C.slot;
    if (C.op == JACC_OP_ALLREDUCE_SUM || C.op == JACC_OP_HALO_EXCHANGE_F32) op.off = C.peer_off;
    else {
        const Buffer &B = g->bufs[C.args[C.op == JACC_OP_ALLGATHER ? 1 : 0].buf];
        op.off = win_off(g, B.dptr, B.bytes);
    }
    return op;
}

// `fuse`: the collective task fused into this kernel (JACC_GRAPH_P2P), or NULL.
// `assign`: a REDUCE's W output was not memset; its kernel stores the sum.
int launch_task(jacc_graph *g, Task &T, cudaStream_t st, int *launches, const Task *fuse = nullptr,
                bool assign = false) {
    jacc_k::PeerOp fop{};
    const jacc_k::PeerOp *fp = nullptr;
    if (fuse) {
        fop = peer_op(g, *fuse);
        fp = &fop;
    }
    auto P = [&](int i) { return g->bufs[T.args[i].buf].dptr; };
    const jacc_schedule_t *sched = T.has_sched ? &T.sched : nullptr;
    const TaskArg *a = T.args.data();
    cudaError_t e = cudaSuccess;
    switch (T.op) {
        case JACC_OP_VADD_F32:
            e = jacc_k::vadd_f32((const float *)P(0), (const float *)P(1), (float *)P(2), (int64_t)a[0].count,
                                 sched, st, launches);
            break;
        case JACC_OP_REDUCE_SUM_F32:
            e = jacc_k::reduce_sum_f32((const float *)P(0), (int64_t)a[0].count, (float *)P(1), T.ws, sched, st,
                                       launches, assign, fp);
            break;
        case JACC_OP_HISTOGRAM_I32:
            e = jacc_k::histogram_i32((const int32_t *)P(0), (int64_t)a[0].count, (int32_t *)P(1),
                                      ((const jacc_hist_params_t *)T.params.data())->nbins, T.ws, sched, st,
                                      launches, fp, assign);
            break;
        case JACC_OP_BLACKSCHOLES_F32:
            e = jacc_k::blackscholes_f32((const float *)P(0), (float *)P(1), (float *)P(2), (int64_t)a[0].count,
                                         sched, st, launches);
            break;
        case JACC_OP_BLACKSCHOLES_SOA_F32:
            e = jacc_k::blackscholes_soa_f32((const float *)P(0), (const float *)P(1), (const float *)P(2),
                                             (const float *)P(3), (const float *)P(4), (float *)P(5),
                                             (float *)P(6), (int64_t)a[0].count, sched, st, launches);
            break;
        case JACC_OP_SGEMM_F32:
            e = jacc_k::sgemm_f32((const float *)P(0), (const float *)P(1), (float *)P(2),
                                  (const jacc_sgemm_params_t *)T.params.data(), T.ws, st, launches);
            break;
        case JACC_OP_NBODY_STEP_F32:
            e = jacc_k::nbody_step_f32((const float4 *)P(0), (int64_t)a[0].count, (float4 *)P(1), (float4 *)P(2),
                                       (int64_t)a[1].count, (const jacc_nbody_params_t *)T.params.data(), T.ws, sched,
                                       st, launches, fp);
            break;
        case JACC_OP_CONV2D_F32: {
            const jacc_conv2d_params_t *cp = (const jacc_conv2d_params_t *)T.params.data();
            const bool halo = cp->flags & JACC_CONV2D_HALO_ROWS;
            e = jacc_k::conv2d_f32((const float *)P(0), cp->H + (halo ? 2 * cp->radius : 0), cp->W,
                                   (const float *)P(1), cp->radius, (float *)P(2), halo ? cp->radius : 0, cp->H, st,
                                   launches);
            break;
        }
        case JACC_OP_CORR_POPC_U32: {
            const jacc_corr_params_t *cp = (const jacc_corr_params_t *)T.params.data();
            e = jacc_k::corr_popc_u32((const uint32_t *)P(0), cp->ta, (const uint32_t *)P(1), cp->tb, cp->words,
                                      (int32_t *)P(2), T.ws, st, launches);
            break;
        }
        case JACC_OP_SPMV_CSR_F32:
            e = jacc_k::spmv_csr_f32((const int32_t *)P(0), (const int32_t *)P(1), (const float *)P(2),
                                     (const float *)P(3), (float *)P(4),
                                     ((const jacc_spmv_params_t *)T.params.data())->n, (int64_t)a[1].count, st,
                                     launches);
            break;
        case JACC_OP_HALO_EXCHANGE_F32: {
            const jacc_halo_params_t *hp = (const jacc_halo_params_t *)T.params.data();
            const float *band = (const float *)P(0);
            float *ext = (float *)P(1);
            const int rk = g->cfg.rank, wd = g->cfg.world;
            if (hp->rows * hp->W == 0 && wd == 1) break;
            if (p2p(g)) {   // peer-memory push + finish (at world 1: the same kernels, no neighbours)
                e = jacc_k::peer_halo(peer_op(g, T), band, ext, hp->rows, hp->W, hp->radius, st, launches);
                break;
            }
            // world 1, or NCCL: band into the middle, zeros past the image,
            // then the neighbours' rows by ncclSend / ncclRecv
            e = jacc_k::halo_local(band, ext, hp->rows, hp->W, hp->radius, rk == 0, rk == wd - 1, st, launches);
            if (e != cudaSuccess || wd == 1) break;
            const uint64_t edge = (uint64_t)hp->radius * hp->W;
            const int r = jacc_nccl::halo_exchange(band, band + (hp->rows * hp->W - edge), ext,
                                                   ext + (hp->rows + hp->radius) * hp->W, edge, rk, wd,
                                                   g->cfg.nccl_comm, st);
            if (r != 0) return fail(JACC_ERR_NCCL, "halo: %s", jacc_nccl::last_error());
            break;
        }
        case JACC_OP_ALLREDUCE_SUM:
        case JACC_OP_ALLGATHER:
        case JACC_OP_BROADCAST: {
            if (p2p(g)) {   // over NVLink peer memory (peer.cu)
                const jacc_k::PeerOp op = peer_op(g, T);
                const int64_t bytes = (int64_t)(a[0].count * dtype_size(a[0].dtype));
                if (T.op == JACC_OP_ALLREDUCE_SUM)
                    e = jacc_k::peer_allreduce(op, P(0), (int64_t)a[0].count, a[0].dtype == JACC_I32, st, launches);
                else if (T.op == JACC_OP_ALLGATHER)
                    e = jacc_k::peer_allgather(op, P(0), bytes, st, launches);
                else
                    e = jacc_k::peer_broadcast(op, ((const jacc_bcast_params_t *)T.params.data())->root, bytes, st,
                                               launches);
                break;
            }
            uint64_t n;
            int dt = nccl_dtype(a[0].dtype, a[0].count, &n);
            if (g->cfg.world == 1 && !g->cfg.nccl_comm) {
                if (T.op == JACC_OP_ALLGATHER && a[0].count)
                    e = cudaMemcpyAsync(P(1), P(0), a[0].count * dtype_size(a[0].dtype), cudaMemcpyDeviceToDevice,
                                        st);
                break;
            }
            int r;
            if (T.op == JACC_OP_ALLREDUCE_SUM)
                r = jacc_nccl::allreduce_sum(P(0), P(0), n, dt, g->cfg.nccl_comm, st);
            else if (T.op == JACC_OP_ALLGATHER)
                r = jacc_nccl::allgather(P(0), P(1), n, dt, g->cfg.nccl_comm, st);
            else
                r = jacc_nccl::broadcast(P(0), P(0), n, dt, ((const jacc_bcast_params_t *)T.params.data())->root,
                                         g->cfg.nccl_comm, st);
            if (r != 0) return fail(JACC_ERR_NCCL, "%s: %s", op_name(T.op), jacc_nccl::last_error());
            break;
        }
        default:
            return fail(JACC_ERR_INVALID_ARG, "op %d", T.op);
    }
    if (e != cudaSuccess) return fail(JACC_ERR_CUDA, "launch %s: %s", op_name(T.op), cudaGetErrorString(e));
    e = cudaGetLastError();
    if (e != cudaSuccess) return fail(JACC_ERR_CUDA, "launch %s: %s", op_name(T.op), cudaGetErrorString(e));
    return JACC_OK;
}

// JACC_GRAPH_MERGE ("merge"): task i = vadd whose output c is the input
// of task i + 1 = reduce, on the same stream, pointers 16-byte aligned ->
// index of the reduce task to fuse with it, else -1.
//
// JACC_GRAPH_P2P (reading R23): task i produces exactly the data that task
// i + 1, a collective, exchanges -> i + 1 is fused into task i's kernel:
//   histogram(keys, bins) [nbins <= 256, n > 0] -> allreduce(bins)
//   reduce(x, out)                              -> allreduce(out)
//   nbody(src, vel, pos_out) [n_tgt > 0]        -> allgather(pos_out -> recv)
int p2p_partner(const jacc_graph *g, int i) {
    const int j = i + 1;
    if (j >= (int)g->tasks.size()) return -1;
    const Task &V = g->tasks[i], &C = g->tasks[j];
    if (C.op == JACC_OP_ALLREDUCE_SUM && V.op == JACC_OP_HISTOGRAM_I32 && C.args[0].buf == V.args[1].buf &&
        ((const jacc_hist_params_t *)V.params.data())->nbins <= 256 && V.args[0].count > 0)
        return j;
    if (C.op == JACC_OP_ALLREDUCE_SUM && V.op == JACC_OP_REDUCE_SUM_F32 && C.args[0].buf == V.args[1].buf) return j;
    if (C.op == JACC_OP_ALLGATHER && V.op == JACC_OP_NBODY_STEP_F32 && C.args[0].buf == V.args[2].buf &&
        V.args[1].count > 0) {
        // The fused finish kernel publishes "ready" (peers may store into
        // the gathered buffer) while its threads still read pos_src[tgt_offset
        // + t].  Safe when the gathered buffer is not pos_src, or when the
        // slots read are this rank's own slot of it (peers write only theirs).
        const int64_t n_tgt = (int64_t)V.args[1].count;
        const int64_t off = ((const jacc_nbody_params_t *)V.params.data())->tgt_offset;
        if (C.args[1].buf != V.args[0].buf || off == (int64_t)g->cfg.rank * n_tgt) return j;
    }
    return -1;
}

int merge_partner(const jacc_graph *g, int i) {
    if ((g->cfg.flags & JACC_GRAPH_NAIVE) || g->cfg.fail_task > 0) return -1;
    if (p2p(g)) {
        const int j = p2p_partner(g, i);
        if (j >= 0) return j;
    }
    if (!(g->cfg.flags & JACC_GRAPH_MERGE)) return -1;
    const int j = i + 1;
    if (j >= (int)g->tasks.size()) return -1;
    const Task &V = g->tasks[i], &R = g->tasks[j];
    if (V.op != JACC_OP_VADD_F32 || R.op != JACC_OP_REDUCE_SUM_F32) return -1;
    if (R.args[0].buf != V.args[2].buf || R.stream != V.stream) return -1;
    auto P = [&](const Task &U, int k) { return (const float *)g->bufs[U.args[k].buf].dptr; };
    return jacc_k::vadd_reduce_fusable(P(V, 0), P(V, 1), P(V, 2)) ? j : -1;
}

// The tasks issued as one kernel with task i (i first): i alone, a merged
// vadd -> reduce pair, a P2P producer -> collective pair, or the triple
// vadd -> reduce -> allreduce (MERGE + P2P).
std::vector<int> fused_group(const jacc_graph *g, int i) {
    std::vector<int> grp{i};
    const int j = merge_partner(g, i);
    if (j < 0) return grp;
    grp.push_back(j);
    if (!is_collective(g->tasks[j].op) && p2p(g) && g->cfg.fail_task == 0) {
        const int k = p2p_partner(g, j);
        if (k >= 0) grp.push_back(k);
    }
    return grp;
}

int issue(jacc_graph *g) {
    const int nb = (int)g->bufs.size(), nt = (int)g->tasks.size();
    std::vector<char> h2d_issued(nb, 0);
    std::vector<char> task_done(nt, 0);
    int launches = 0;
    jacc_stats_t &S = g->stats;
    const bool naive = g->cfg.flags & JACC_GRAPH_NAIVE;
    const bool timing = !(g->cfg.flags & JACC_GRAPH_NO_TIMING);
    // pre-pass: kernel groups (merges), then which tasks' dependency events
    // some other stream waits on -- only those are recorded
    std::vector<std::vector<int>> group(nt);
    for (Task &T : g->tasks) T.fused_into = -1;
    for (const Action &A : g->plan) {
        if ((A.kind != A_KERNEL && A.kind != A_COLLECTIVE) || g->tasks[A.task].fused_into >= 0 ||
            !group[A.task].empty())
            continue;
        group[A.task] = fused_group(g, A.task);
        for (size_t k = 1; k < group[A.task].size(); ++k) g->tasks[group[A.task][k]].fused_into = A.task;
    }
    std::vector<char> need_dep(nt, 0);
    for (int t = 0; t < nt; ++t) {
        if (group[t].empty()) continue;
        cudaStream_t st = stream_of(g, g->tasks[t]);
        for (int u : group[t])
            for (int p : g->tasks[u].preds)
                if (g->tasks[p].fused_into != t && p != t && stream_of(g, g->tasks[p]) != st) need_dep[p] = 1;
    }
    for (const Action &A : g->plan)
        if (A.kind == A_D2H && stream_of(g, g->tasks[A.task]) != g->d2h) need_dep[A.task] = 1;

    if (!naive) {   // all H2D first, critical path first; kernels wait on their own events
        for (int i : g->h2d_order) {
            Buffer &B = g->bufs[g->plan[i].buf];
            CK(cudaMemcpyAsync(B.dptr, (const void *)B.host, B.bytes, cudaMemcpyHostToDevice, g->h2d));
            CK(cudaEventRecord(B.ev_h2d, g->h2d));
            h2d_issued[g->plan[i].buf] = 1;
        }
    }
    for (size_t ai = 0; ai < g->plan.size(); ++ai) {
        const Action &A = g->plan[ai];
        if (A.kind == A_H2D) {
            if (!naive) continue;
            Buffer &B = g->bufs[A.buf];
            CK(cudaMemcpyAsync(B.dptr, (const void *)B.host, B.bytes, cudaMemcpyHostToDevice, g->h2d));
            CK(cudaEventRecord(B.ev_h2d, g->h2d));
            h2d_issued[A.buf] = 1;
        } else if (A.kind == A_KERNEL || A.kind == A_COLLECTIVE) {
            if (task_done[A.task]) continue;   // issued inside an earlier merged kernel
            Task &T = g->tasks[A.task];
            if (g->cfg.fail_task > 0 && A.task == g->cfg.fail_task - 1)
                return fail(JACC_ERR_INJECTED, "failure injected at task %d", A.task);
            cudaStream_t st = stream_of(g, T);
            const std::vector<int> &grp = group[A.task];
            // timing events: under CUDA-graph capture they must be EXTERNAL
            // record nodes (a plain record is only a capture dependency)
            auto rec = [&](cudaEvent_t e) {
                return g->capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
            };
            for (int t : grp) {
                const Task &U = g->tasks[t];
                for (const TaskArg &a : U.args)
                    if (h2d_issued[a.buf] && g->h2d != st) CK(cudaStreamWaitEvent(st, g->bufs[a.buf].ev_h2d, 0));
                for (int p : U.preds) {
                    const Task &Pt = g->tasks[p];
                    if (p != A.task && Pt.fused_into != A.task && stream_of(g, Pt) != st)
                        CK(cudaStreamWaitEvent(st, Pt.ev_dep, 0));
                }
            }
            if (timing)
                for (int t : grp) CK(rec(g->tasks[t].ev_start));
            // MEMSET0 actions (auto-zero of @Atomic outputs) of the
            // group's tasks; a reduction's sum and a histogram's bins are
            // instead assigned (not added) by their kernels' last block --
            // one memset node less per task
            bool assign = false;
            for (int t : grp)
                for (int b : g->memset_bufs[t]) {
                    if (g->tasks[t].op == JACC_OP_REDUCE_SUM_F32 || g->tasks[t].op == JACC_OP_HISTOGRAM_I32) {
                        assign = true;
                        continue;
                    }
                    CK(cudaMemsetAsync(g->bufs[b].dptr, 0, g->bufs[b].bytes, st));
                }
            int rc;
            const Task *coll = grp.size() > 1 && is_collective(g->tasks[grp.back()].op) ? &g->tasks[grp.back()] : nullptr;
            if (grp.size() > 1 && g->tasks[grp[1]].op == JACC_OP_REDUCE_SUM_F32 && T.op == JACC_OP_VADD_F32) {
                const Task &Rt = g->tasks[grp[1]];
                auto P = [&](const Task &U, int i) { return g->bufs[U.args[i].buf].dptr; };
                jacc_k::PeerOp op{};
                if (coll) op = peer_op(g, *coll);
                cudaError_t e = jacc_k::vadd_reduce_f32(
                    (const float *)P(T, 0), (const float *)P(T, 1), (float *)P(T, 2), (int64_t)T.args[0].count,
                    (float *)P(Rt, 1), Rt.ws, Rt.has_sched ? &Rt.sched : nullptr, st, &launches, assign,
                    coll ? &op : nullptr);
                rc = e == cudaSuccess ? JACC_OK : fail(JACC_ERR_CUDA, "launch vadd+reduce: %s", cudaGetErrorString(e));
            } else {
                rc = launch_task(g, T, st, &launches, coll, assign);
            }
            if (rc != JACC_OK) return rc;
            for (int t : grp) {
                if (timing) CK(rec(g->tasks[t].ev_end));
                if (need_dep[t]) CK(cudaEventRecord(g->tasks[t].ev_dep, st));   // cross-stream dependency marker
                task_done[t] = 1;
            }
        } else if (A.kind == A_D2H) {
            Buffer &B = g->bufs[A.buf];
            const Task &W = g->tasks[A.task];
            cudaStream_t ws = stream_of(g, W);
            if (ws != g->d2h) CK(cudaStreamWaitEvent(g->d2h, W.ev_dep, 0));
            CK(cudaMemcpyAsync((void *)B.host, B.dptr, B.bytes, cudaMemcpyDeviceToHost, g->d2h));
        }
        // A_MEMSET0 is issued with its task's kernel (same stream)
    }
    S.launches = (uint64_t)launches;
    return JACC_OK;
}

int sync_all(jacc_graph *g) {
    cudaError_t first = cudaSuccess;
    auto chk = [&](cudaError_t e) { if (e != cudaSuccess && first == cudaSuccess) first = e; };
    if (g->last_was_replay) {   // the graph launch joined every stream into compute[0]
        chk(cudaStreamSynchronize(g->compute[0]));
    } else {
        for (int i = 0; i < g->n_streams; ++i) chk(cudaStreamSynchronize(g->compute[i]));
        if (g->h2d) chk(cudaStreamSynchronize(g->h2d));
        if (g->comm && g->comm != g->h2d) chk(cudaStreamSynchronize(g->comm));
        if (g->d2h && g->d2h != g->h2d) chk(cudaStreamSynchronize(g->d2h));
    }
    if (first != cudaSuccess) return cuda_fail(first, "sync");
    return JACC_OK;
}

bool same_plan(const std::vector<Action> &a, const std::vector<Action> &b) {
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (a[i].kind != b[i].kind || a[i].buf != b[i].buf || a[i].task != b[i].task) return false;
    return true;
}

// SURVEY §8(f) f2, "plan replay": the first execute of a plan issues its
// actions under CUDA stream capture (every graph stream forked from
// compute[0] and joined back), later executes with an identical plan launch
// the instantiated graph -- one launch instead of one per copy, memset,
// kernel, event and collective.  Plans that cannot be captured (pageable
// host memory) are remembered and issued directly.
int issue_replay(jacc_graph *g) {
    cudaStream_t origin = g->compute[0];
    if (g->exec && same_plan(g->exec_plan, g->plan)) {
        CK(cudaGraphLaunch(g->exec, origin));
        g->stats.launches = g->exec_launches;
        g->stats.graph_replays++;
        return JACC_OK;
    }
    if (g->exec_failed && same_plan(g->exec_plan, g->plan)) return issue(g);
    if (g->exec) {
        cudaGraphExecDestroy(g->exec);
        g->exec = nullptr;
    }
    std::vector<cudaStream_t> others;
    for (int i = 1; i < g->n_streams; ++i) others.push_back(g->compute[i]);
    for (cudaStream_t s : {g->h2d, g->d2h, g->comm})
        if (s && s != origin && std::find(others.begin(), others.end(), s) == others.end()) others.push_back(s);
    if (!g->ev_fork) CK(cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming));
    while (g->ev_join.size() < others.size()) {
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        g->ev_join.push_back(e);
    }
    CK(cudaStreamBeginCapture(origin, cudaStreamCaptureModeRelaxed));
    cudaError_t e = cudaEventRecord(g->ev_fork, origin);
    for (size_t i = 0; e == cudaSuccess && i < others.size(); ++i) e = cudaStreamWaitEvent(others[i], g->ev_fork, 0);
    g->capturing = true;
    int rc = e == cudaSuccess ? issue(g) : cuda_fail(e, "capture fork");
    g->capturing = false;
    for (size_t i = 0; rc == JACC_OK && i < others.size(); ++i) {
        e = cudaEventRecord(g->ev_join[i], others[i]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(origin, g->ev_join[i], 0);
        if (e != cudaSuccess) rc = cuda_fail(e, "capture join");
    }
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(origin, &graph);
    if (rc == JACC_OK && e == cudaSuccess && graph)
        e = cudaGraphInstantiate(&g->exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    g->exec_plan = g->plan;
    if (rc != JACC_OK || e != cudaSuccess || !g->exec) {
        // not capturable (e.g. pageable memcpy): clear the error, issue directly
        cudaGetLastError();
        if (g->exec) { cudaGraphExecDestroy(g->exec); g->exec = nullptr; }
        g->exec_failed = true;
        return issue(g);
    }
    g->exec_failed = false;
    g->exec_launches = g->stats.launches;
    g->stats.graph_captures++;
    CK(cudaGraphLaunch(g->exec, origin));
    return JACC_OK;
}

int peer_init_window(jacc_graph *g, size_t bytes) {
    if (bytes == 0) bytes = (size_t)64 << 20;
    if (bytes < jacc_k::kPeerHeaderBytes + 4096) bytes = jacc_k::kPeerHeaderBytes + 4096;
    int rc = ensure_resources(g);
    if (rc != JACC_OK) return rc;
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return fail(JACC_ERR_OOM, "P2P window of %zu bytes", bytes);
    }
    CK(cudaMemset(p, 0, bytes));   // flags, counts and tickets start at 0
    g->win = (char *)p;
    g->win_bytes = bytes;
    g->win_top = jacc_k::kPeerHeaderBytes;
    return JACC_OK;
}

}  // namespace

// ================================================================ ABI
extern "C" {

const char *jacc_status_string(int s) {
    switch (s) {
        case JACC_OK: return "JACC_OK";
        case JACC_ERR_INVALID_ARG: return "JACC_ERR_INVALID_ARG";
        case JACC_ERR_STATE: return "JACC_ERR_STATE";
        case JACC_ERR_ACCESS: return "JACC_ERR_ACCESS";
        case JACC_ERR_ALIAS: return "JACC_ERR_ALIAS";
        case JACC_ERR_DEVICE: return "JACC_ERR_DEVICE";
        case JACC_ERR_OOM: return "JACC_ERR_OOM";
        case JACC_ERR_CUDA: return "JACC_ERR_CUDA";
        case JACC_ERR_NCCL: return "JACC_ERR_NCCL";
        case JACC_ERR_NOT_FOUND: return "JACC_ERR_NOT_FOUND";
        case JACC_ERR_UNSUPPORTED: return "JACC_ERR_UNSUPPORTED";
        case JACC_ERR_INJECTED: return "JACC_ERR_INJECTED";
        default: return "JACC_ERR_?";
    }
}

const char *jacc_last_error(void) { return g_last_error.c_str(); }

int jacc_abi_version(void) { return JACC_ABI_VERSION; }

size_t jacc_abi_sizeof(const char *name) {
    if (!name) return 0;
#define S(T) if (!strcmp(name, #T)) return sizeof(T)
    S(jacc_arg_t); S(jacc_schedule_t); S(jacc_config_t); S(jacc_stats_t);
    S(jacc_hist_params_t); S(jacc_sgemm_params_t); S(jacc_nbody_params_t); S(jacc_bcast_params_t);
    S(jacc_conv2d_params_t); S(jacc_corr_params_t); S(jacc_spmv_params_t); S(jacc_peer_handle_t);
    S(jacc_halo_params_t);
#undef S
    return 0;
}

int jacc_graph_create(jacc_graph_t **out, const jacc_config_t *cfg) {
    if (!out || !cfg) return fail(JACC_ERR_INVALID_ARG, "NULL argument");
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
        return fail(JACC_ERR_INVALID_ARG, "rank %d / world %d", cfg->rank, cfg->world);
    if (cfg->n_compute < 0 || cfg->n_compute > JACC_MAX_STREAMS)
        return fail(JACC_ERR_INVALID_ARG, "n_compute %d", cfg->n_compute);
    if (cfg->world > 1 && !cfg->nccl_comm && !(cfg->flags & JACC_GRAPH_P2P))
        return fail(JACC_ERR_INVALID_ARG, "world > 1 needs an NCCL communicator (or JACC_GRAPH_P2P)");
    if ((cfg->flags & JACC_GRAPH_P2P) && cfg->world > JACC_PEER_MAX)
        return fail(JACC_ERR_INVALID_ARG, "JACC_GRAPH_P2P: world %d > %d", cfg->world, JACC_PEER_MAX);
    if (cfg->device < 0) return fail(JACC_ERR_INVALID_ARG, "device %d", cfg->device);
    if ((cfg->alloc == nullptr) != (cfg->free == nullptr))
        return fail(JACC_ERR_INVALID_ARG, "alloc and free hooks come together");
    jacc_graph *g = new (std::nothrow) jacc_graph();
    if (!g) return fail(JACC_ERR_OOM, "host allocation");
    g->cfg = *cfg;
    memset(&g->stats, 0, sizeof g->stats);
    *out = g;
    return JACC_OK;
}

int jacc_graph_add_task(jacc_graph_t *g, jacc_op_t op, const jacc_arg_t *args, int nargs, const void *params,
                        size_t params_size, const jacc_schedule_t *sched, int device, int *task_id) {
    if (!g || (nargs > 0 && !args) || nargs < 0) return fail(JACC_ERR_INVALID_ARG, "NULL argument");
    if (g->state == ST_EXECUTING) return fail(JACC_ERR_STATE, "graph is executing");
    if (device != g->cfg.device)
        return fail(JACC_ERR_DEVICE, "task device %d != graph device %d (one process per GPU)", device,
                    g->cfg.device);
    int rc = validate(g, op, args, nargs, params, params_size);
    if (rc != JACC_OK) return rc;
    Task T;
    T.op = op;
    std::vector<Buffer> newbufs;
    for (int i = 0; i < nargs; ++i) {
        int id = -1;
        rc = resolve_buffer(g, args[i], newbufs, &id);
        if (rc != JACC_OK) return rc;
        T.args.push_back({id, args[i].count, args[i].dtype, args[i].access, args[i].flags});
    }
    // a written buffer may not appear twice in one task (in-place aliasing)
    for (size_t i = 0; i < T.args.size(); ++i)
        for (size_t j = 0; j < T.args.size(); ++j)
            if (i != j && T.args[i].buf == T.args[j].buf && (T.args[i].access & JACC_WRITE))
                return fail(JACC_ERR_ALIAS, "arg %zu (written) aliases arg %zu", i, j);
    if (params && params_size) T.params.assign((const unsigned char *)params, (const unsigned char *)params + params_size);
    if (sched) { T.sched = *sched; T.has_sched = true; }
    else memset(&T.sched, 0, sizeof T.sched);
    for (Buffer &b : newbufs) g->bufs.push_back(b);
    for (const TaskArg &a : T.args)
        if (a.flags & JACC_ARG_CACHABLE) g->bufs[a.buf].cachable = true;
    // dependency inference (reading R9)
    const int t = (int)g->tasks.size();
    for (int i = 0; i < t; ++i) {
        bool edge = false;
        for (const TaskArg &x : g->tasks[i].args)
            for (const TaskArg &y : T.args)
                if (x.buf == y.buf && ((x.access & JACC_WRITE) || (y.access & JACC_WRITE))) edge = true;
        if (edge) T.preds.push_back(i);
    }
    g->tasks.push_back(std::move(T));
    g->planned = false;
    if (g->state == ST_DONE || g->state == ST_FAILED) g->state = ST_BUILDING;
    if (task_id) *task_id = t;
    return JACC_OK;
}

// A failed execute may have run some kernels already: the device copies of
// the buffers they wrote (e.g. a CACHABLE RW velocity in an N-body chain) no
// longer equal the host values, which a failure leaves untouched (R8).  Drop
// every residency claim so the next execute re-uploads from the host.
static void drop_residency(jacc_graph *g) {
    for (Buffer &B : g->bufs)
        if (!B.device) B.dev_current = false;
    g->planned = false;
}

// JACC_LOG=1: host-side phase times of every execute on stderr (issue
// latency diagnostics; nothing is logged otherwise).
static bool log_on() {
    static const bool on = [] { const char *e = getenv("JACC_LOG"); return e && e[0] == '1'; }();
    return on;
}
static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// NVTX range for the scope of an ABI call (a no-op unless a tool injects NVTX)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

int jacc_graph_execute(jacc_graph_t *g) {
    NvtxRange nvtx("jacc_graph_execute");
    if (!g) return fail(JACC_ERR_INVALID_ARG, "NULL graph");
    if (g->state == ST_EXECUTING) return fail(JACC_ERR_STATE, "graph is already executing");
    const double t0 = log_on() ? now_us() : 0.0;
    ensure_plan(g);
    const double t1 = log_on() ? now_us() : 0.0;
    int rc = ensure_resources(g);
    const double t2 = log_on() ? now_us() : 0.0;
    if (rc == JACC_OK) rc = prepare_memory(g);
    if (log_on())
        fprintf(stderr, "[jacc] execute: plan %.1f us, resources %.1f us, memory %.1f us\n", t1 - t0, t2 - t1,
                now_us() - t2);
    if (rc != JACC_OK) { drop_residency(g); g->state = ST_FAILED; return rc; }
    ensure_plan(g);   // a device copy (re)allocated just now is not resident
    plan_counts(g, &g->stats);
    g->have_times = false;
    g->state = ST_EXECUTING;
    g->last_was_replay = false;
    if ((g->cfg.flags & JACC_GRAPH_REPLAY) && !(g->cfg.flags & JACC_GRAPH_NAIVE) && g->cfg.fail_task == 0) {
        const uint64_t before = g->stats.graph_replays + g->stats.graph_captures;
        rc = issue_replay(g);
        g->last_was_replay = rc == JACC_OK && g->stats.graph_replays + g->stats.graph_captures > before;
    } else {
        const double t3 = log_on() ? now_us() : 0.0;
        rc = issue(g);
        if (log_on()) fprintf(stderr, "[jacc] execute: issue %.1f us (%zu actions)\n", now_us() - t3, g->plan.size());
    }
    if (rc != JACC_OK) {
        sync_all(g);   // drain what was issued; no D2H after the failure point
        drop_residency(g);
        g->state = ST_FAILED;
        g->pending_error = rc;
        return rc;
    }
    return JACC_OK;
}

int jacc_graph_sync(jacc_graph_t *g) {
    NvtxRange nvtx("jacc_graph_sync");
    if (!g) return fail(JACC_ERR_INVALID_ARG, "NULL graph");
    if (g->state != ST_EXECUTING) {
        if (g->state == ST_FAILED) return g->pending_error ? g->pending_error : JACC_ERR_STATE;
        return JACC_OK;
    }
    int rc = sync_all(g);
    if (rc != JACC_OK) {
        drop_residency(g);
        g->state = ST_FAILED;
        g->pending_error = rc;
        return rc;
    }
    if (!(g->cfg.flags & JACC_GRAPH_NO_TIMING)) {
        for (Task &T : g->tasks) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, T.ev_start, T.ev_end) == cudaSuccess) T.ms = ms;
        }
        g->have_times = true;
    }
    for (Buffer &B : g->bufs) {
        if (!B.device) {
            B.dev_current = true;
            B.invalidated = false;
        }
    }
    jacc_stats_t &S = g->stats;
    S.total_h2d_count += S.h2d_count;
    S.total_h2d_bytes += S.h2d_bytes;
    S.total_d2h_count += S.d2h_count;
    S.total_d2h_bytes += S.d2h_bytes;
    S.total_kernels += S.kernels;
    S.total_collectives += S.collectives;
    S.total_launches += S.launches;
    S.executes += 1;
    g->state = ST_DONE;
    g->pending_error = JACC_OK;
    return JACC_OK;
}

int jacc_graph_stats(const jacc_graph_t *g, jacc_stats_t *out) {
    if (!g || !out) return fail(JACC_ERR_INVALID_ARG, "NULL argument");
    jacc_graph *gm = const_cast<jacc_graph *>(g);
    if (gm->state != ST_EXECUTING) {
        if (!gm->planned) make_plan(gm);
        if (gm->state == ST_BUILDING) plan_counts(gm, &gm->stats);
    }
    *out = g->stats;
    out->n_tasks = (int32_t)g->tasks.size();
    out->n_buffers = (int32_t)g->bufs.size();
    out->state = g->state;
    return JACC_OK;
}

int jacc_graph_task_ms(const jacc_graph_t *g, int task_id, float *ms) {
    if (!g || !ms) return fail(JACC_ERR_INVALID_ARG, "NULL argument");
    if (task_id < 0 || task_id >= (int)g->tasks.size()) return fail(JACC_ERR_NOT_FOUND, "task %d", task_id);
    if (g->cfg.flags & JACC_GRAPH_NO_TIMING) return fail(JACC_ERR_STATE, "graph created with JACC_GRAPH_NO_TIMING");
    if (!g->have_times) return fail(JACC_ERR_STATE, "no completed execute");
    *ms = g->tasks[task_id].ms;
    return JACC_OK;
}

int jacc_graph_set_fail_task(jacc_graph_t *g, int32_t fail_task) {
    if (!g || fail_task < 0) return fail(JACC_ERR_INVALID_ARG, "NULL graph or fail_task < 0");
    if (g->state == ST_EXECUTING) return fail(JACC_ERR_STATE, "graph is executing");
    g->cfg.fail_task = fail_task;
    g->planned = false;   // merge / fusion decisions depend on the hook
    return JACC_OK;
}

int jacc_graph_dump(jacc_graph_t *g, char *buf, size_t cap, size_t *needed) {
    if (!g) return fail(JACC_ERR_INVALID_ARG, "NULL graph");
    if (g->state != ST_EXECUTING) make_plan(g);
    std::string s = dump_text(g);
    if (needed) *needed = s.size() + 1;
    if (buf) {
        if (cap == 0) return fail(JACC_ERR_INVALID_ARG, "cap 0");
        size_t n = std::min(cap - 1, s.size());
        memcpy(buf, s.data(), n);
        buf[n] = 0;
        if (n < s.size()) return fail(JACC_ERR_INVALID_ARG, "cap %zu < %zu", cap, s.size() + 1);
    }
    return JACC_OK;
}

int jacc_buffer_invalidate(jacc_graph_t *g, const void *host_ptr) {
    if (!g) return fail(JACC_ERR_INVALID_ARG, "NULL graph");
    if (g->state == ST_EXECUTING) return fail(JACC_ERR_STATE, "graph is executing");
    for (Buffer &B : g->bufs)
        if (B.host == (uintptr_t)host_ptr && !B.device) {
            B.invalidated = true;
            g->planned = false;
            return JACC_OK;
        }
    return fail(JACC_ERR_NOT_FOUND, "no host buffer at %p", host_ptr);
}

int jacc_peer_init(jacc_graph_t *g, size_t window_bytes, jacc_peer_handle_t *out) {
    if (!g || !out) return fail(JACC_ERR_INVALID_ARG, "NULL argument");
    if (!(g->cfg.flags & JACC_GRAPH_P2P)) return fail(JACC_ERR_STATE, "not a JACC_GRAPH_P2P graph");
    if (g->win) return fail(JACC_ERR_STATE, "peer window already initialised");
    int rc = peer_init_window(g, window_bytes);
    if (rc != JACC_OK) return rc;
    memset(out, 0, sizeof *out);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, g->win));
    static_assert(sizeof h <= sizeof out->ipc, "ipc handle size");
    memcpy(out->ipc, &h, sizeof h);
    out->window_bytes = g->win_bytes;
    out->rank = g->cfg.rank;
    out->device = g->cfg.device;
    return JACC_OK;
}

int jacc_peer_connect(jacc_graph_t *g, const jacc_peer_handle_t *h, int n) {
    if (!g || !h) return fail(JACC_ERR_INVALID_ARG, "NULL argument");
    if (!g->win) return fail(JACC_ERR_STATE, "jacc_peer_init first");
    if (g->peer_connected) return fail(JACC_ERR_STATE, "already connected");
    if (n != g->cfg.world) return fail(JACC_ERR_INVALID_ARG, "%d handles for world %d", n, g->cfg.world);
    for (int q = 0; q < n; ++q) {
        if (h[q].rank != q) return fail(JACC_ERR_INVALID_ARG, "handle %d is rank %d's", q, h[q].rank);
        if (h[q].window_bytes != g->win_bytes)
            return fail(JACC_ERR_INVALID_ARG, "window sizes differ (rank %d: %llu, here %zu)", q,
                        (unsigned long long)h[q].window_bytes, g->win_bytes);
    }
    CK(cudaSetDevice(g->cfg.device));
    for (int q = 0; q < n; ++q) {
        if (q == g->cfg.rank) continue;
        cudaIpcMemHandle_t ih;
        memcpy(&ih, h[q].ipc, sizeof ih);
        void *p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            for (int k = 0; k < q; ++k)
                if (g->peer_base[k]) { cudaIpcCloseMemHandle(g->peer_base[k]); g->peer_base[k] = nullptr; }
            return cuda_fail(e, "cudaIpcOpenMemHandle (peer window)");
        }
        g->peer_base[q] = (char *)p;
    }
    g->peer_connected = true;
    return JACC_OK;
}

int jacc_peer_alloc(jacc_graph_t *g, size_t bytes, void **dptr) {
    if (!g || !dptr) return fail(JACC_ERR_INVALID_ARG, "NULL argument");
    if (!g->win) {
        if (!(g->cfg.flags & JACC_GRAPH_P2P) || g->cfg.world > 1)
            return fail(JACC_ERR_STATE, "no peer window (JACC_GRAPH_P2P + jacc_peer_init)");
        int rc = peer_init_window(g, 0);
        if (rc != JACC_OK) return rc;
    }
    const int64_t off = win_alloc(g, bytes);
    if (off < 0) return fail(JACC_ERR_OOM, "P2P window full (%zu bytes requested)", bytes);
    *dptr = g->win + off;
    return JACC_OK;
}

int jacc_graph_destroy(jacc_graph_t *g) {
    if (!g) return JACC_OK;
    if (g->res_ready) {
        cudaSetDevice(g->cfg.device);
        sync_all(g);
        // JACC_GRAPH_P2P: wait until every rank has reached destroy before this
        // window is freed -- a slower peer may still owe it a flag store
        // (e.g. a broadcast's "ready" that no rank waits for)
        if (g->peer_connected && g->cfg.world > 1 && g->state != ST_FAILED &&
            jacc_k::peer_barrier(peer_ctx(g), jacc_k::kPeerBarrierSlot, g->compute[0]) == cudaSuccess)
            cudaStreamSynchronize(g->compute[0]);
        for (Buffer &B : g->bufs) {
            if (!B.device && !B.in_window) dev_free(g, B.dptr, B.bytes);
            if (B.ev_h2d) cudaEventDestroy(B.ev_h2d);
        }
        for (Task &T : g->tasks) {
            dev_free(g, T.ws, T.ws_bytes);
            if (T.ev_start) cudaEventDestroy(T.ev_start);
            if (T.ev_end) cudaEventDestroy(T.ev_end);
            if (T.ev_dep) cudaEventDestroy(T.ev_dep);
        }
        if (g->own_compute)
            for (int i = 0; i < g->n_streams; ++i) cudaStreamDestroy(g->compute[i]);
        if (g->own_h2d) cudaStreamDestroy(g->h2d);
        if (g->own_d2h) cudaStreamDestroy(g->d2h);
        if (g->own_comm) cudaStreamDestroy(g->comm);
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->ev_fork) cudaEventDestroy(g->ev_fork);
        for (cudaEvent_t e : g->ev_join) cudaEventDestroy(e);
    }
    for (int q = 0; q < JACC_PEER_MAX; ++q)
        if (g->peer_base[q]) cudaIpcCloseMemHandle(g->peer_base[q]);
    if (g->win) cudaFree(g->win);
    delete g;
    return JACC_OK;
}

}  // extern "C"
