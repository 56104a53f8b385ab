/*
 * jacc.h -- C ABI of libjacc.so, the B200-native (sm_100a) Jacc task-graph
 * runtime and its hand-written CUDA kernels.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section in brackets);
 * SURVEY §8(b) is the boundary table this header implements; DESIGN.md
 * lists every reading (R1..R20) of a silent or ambiguous passage.
 *
 * Model (§2, §2.3):
 *   - a TASK is "a method reference, a parameter list and some scheduling
 *     metadata" (P:86 [§2]) -> jacc_graph_add_task(op, args, params,
 *     schedule, device);
 *   - tasks are "mapped onto hardware when they are inserted into a task
 *     graph" -> the `device` argument, cf. executeTaskOn;
 *   - the TASK GRAPH is a DAG; the runtime "infer[s] all the data
 *     dependencies between tasks" (P:289 [§2.3]) from the per-argument
 *     @Read/@Write/@ReadWrite access (Table 1);
 *   - each task is lowered to data transfers, execution and sync (P:93-94,
 *     P:288); redundant transfers are eliminated and independent kernels
 *     are issued out of order (P:61 [§1]);
 *   - `execute` "blocks until either all tasks ... have completed or an
 *     exception occurs" and makes "all outstanding updates to the host
 *     memory ... visible" (P:169-171 [§2.1.2]).  Here that is
 *     jacc_graph_execute (asynchronous issue) + jacc_graph_sync (block,
 *     commit); the paper's blocking execute == execute followed by sync.
 *   - the graph executes atomically: the host must not touch bound host
 *     buffers between execute and sync (P:214 [§2.2.2], P:375 [§3.2.1]).
 *
 * Conventions for every entry point:
 *   - returns a jacc_status_t (0 == JACC_OK).  No C++ exception, abort or
 *     exit ever crosses the ABI; the detail of the last error of the
 *     calling thread is jacc_last_error().
 *   - pointers are plain host or device pointers; sizes are element counts
 *     unless the name says bytes.  No torch type appears here.
 *   - a graph is confined to one host thread at a time.
 */
#ifndef JACC_H_
#define JACC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JACC_ABI_VERSION 2
#define JACC_MAX_STREAMS 8
#define JACC_PEER_MAX 8     /* ranks of one NVLink/NVSwitch domain (JACC_GRAPH_P2P) */

/* ------------------------------------------------------------ status codes */
typedef enum jacc_status {
    JACC_OK = 0,
    JACC_ERR_INVALID_ARG = 1,  /* NULL/size/dtype/param error              */
    JACC_ERR_STATE = 2,        /* call not allowed in the graph's state     */
    JACC_ERR_ACCESS = 3,       /* access mode not allowed by the op        */
    JACC_ERR_ALIAS = 4,        /* host ranges partially overlap            */
    JACC_ERR_DEVICE = 5,       /* task device != graph device              */
    JACC_ERR_OOM = 6,          /* device allocation failed                 */
    JACC_ERR_CUDA = 7,         /* CUDA runtime/driver error                */
    JACC_ERR_NCCL = 8,         /* NCCL missing or failed                   */
    JACC_ERR_NOT_FOUND = 9,    /* unknown buffer / task id                 */
    JACC_ERR_UNSUPPORTED = 10, /* shape/size the kernels do not support     */
    JACC_ERR_INJECTED = 11     /* test hook: failure injected at a task    */
} jacc_status_t;

/* ---------------------------------------------------- element types (R1) */
typedef enum jacc_dtype {
    JACC_F32 = 1,   /* 4-byte IEEE binary32 */
    JACC_I32 = 2,   /* 4-byte two's complement */
    JACC_F32X4 = 3  /* 16-byte {x, y, z, w} binary32, 16-byte aligned on device */
} jacc_dtype_t;

/* ------------------------- per-argument access, Table 1 */
#define JACC_READ 1u       /* @Read:      input only                      */
#define JACC_WRITE 2u      /* @Write:     output only (fully overwritten, or
                              auto-zeroed when the op's output is @Atomic) */
#define JACC_READWRITE 3u  /* @ReadWrite: input and output                */

/* ------------------------------------------------- per-argument flags */
#define JACC_ARG_DEVICE 1u   /* ptr is a caller-owned DEVICE pointer: used in
                                place, never transferred (R5)   */
#define JACC_ARG_CACHABLE 2u /* Table 1 `cachable`, reading R5:
                                the device copy may stay resident across
                                executes; after the host writes the buffer,
                                call jacc_buffer_invalidate()               */

/* ------------------------------------------------------- graph flags */
#define JACC_GRAPH_NAIVE 1u  /* no transfer elision (SPEC S:425 naive
                                lowering), all actions on one stream: the
                                counted-copies comparison baseline         */
#define JACC_GRAPH_SERIAL 2u /* one compute stream (no out-of-order issue)   */
#define JACC_GRAPH_REPLAY 4u /* plan replay: the issued
                                action list is captured once into a CUDA
                                graph and re-launched by later executes with
                                the same plan (one launch instead of one per
                                action).  A plan that cannot be captured
                                (e.g. pageable host memory) is issued
                                directly; stats.graph_captures/replays say
                                which happened                              */
#define JACC_GRAPH_MERGE 8u  /* task merge ("eliminate, merge and
                                re-organize"): a vadd task
                                immediately followed by a reduce task of its
                                output on the same stream is issued as ONE
                                fused kernel (c written, its sum taken in the
                                same pass, bit-identical to the pair); the
                                action list and counted copies are unchanged,
                                both tasks report the fused kernel's time   */
#define JACC_GRAPH_P2P 16u   /* collectives over NVLink peer memory instead of
                                NCCL (reading R23): every rank maps the other
                                ranks' symmetric window (jacc_peer_init /
                                jacc_peer_connect) and the collective's data
                                moves as plain stores into peer memory.  A
                                collective task that directly follows the
                                kernel producing its data is FUSED into that
                                kernel (histogram -> allreduce(bins), reduce
                                -> allreduce(out), N-body step ->
                                allgather(pos_out)): each block pushes its
                                results to the peers as it finishes them and
                                the last block completes the exchange -- one
                                kernel, no NCCL.  Other collective tasks run
                                as standalone peer-memory kernels.  Every
                                rank must build the same graph (SPMD), as for
                                NCCL; no communicator is needed.  With
                                JACC_GRAPH_MERGE as well, vadd -> reduce ->
                                allreduce is one kernel.  Limits: world <=
                                JACC_PEER_MAX, 1023 collective tasks per
                                graph; a peer that never arrives makes the
                                waiting kernel trap after 30 s (sync then
                                returns JACC_ERR_CUDA) instead of hanging.  */
#define JACC_GRAPH_NO_TIMING 32u /* no per-task timing events (jacc_graph_task_ms
                                then fails with _STATE): for many-task graphs
                                whose cost is the events, e.g. the paper's
                                K-iteration protocol            */

/* -------------------------------------------------------------- ops */
typedef enum jacc_op {
    /* c[i] = a[i] + b[i].  args: a:R f32[n], b:R f32[n], c:W f32[n].
     * Vector Addition, P:476-477 [§4.2].  Map; HBM-bound, 12 B/element.   */
    JACC_OP_VADD_F32 = 1,
    /* out[0] (+)= sum_i x[i].  args: x:R f32[n], out:W|RW f32[1].
     * Reduction, P:130-141 [§2.1.2] and P:479: an @Atomic(op=ADD) field,
     * auto-zeroed in W mode.  Deterministic single-pass tree.      */
    JACC_OP_REDUCE_SUM_F32 = 2,
    /* bins[k] (+)= #{i : keys[i] == k}, 0 <= k < nbins; out-of-range keys
     * are ignored (R11).  args: keys:R i32[n], bins:W|RW i32[nbins];
     * params jacc_hist_params_t.  Histogram; @Atomic.   */
    JACC_OP_HISTOGRAM_I32 = 3,
    /* APARAPI Black-Scholes (formula = reading R12).  args:
     * rand:R f32[n] (u in [0,1)), call:W f32[n], put:W f32[n].            */
    JACC_OP_BLACKSCHOLES_F32 = 4,
    /* Same pricing with explicit parameters (parity coverage of ln(S/K)!=0).
     * args: S,K,T,R,sigma:R f32[n], call:W f32[n], put:W f32[n].          */
    JACC_OP_BLACKSCHOLES_SOA_F32 = 5,
    /* C = A.B, row-major, beta = 0 (reading R13).
     * args: A:R f32[M*lda], B:R f32[K*ldb], C:W f32[M*ldc];
     * params jacc_sgemm_params_t.  Only the M x N window of C is written; as
     * for every W argument (never uploaded), the rest of the buffer is
     * undefined after execute.                                              */
    JACC_OP_SGEMM_F32 = 6,
    /* One symplectic-Euler step of softened direct-sum gravity (north_star;
     * not in the paper, reading R16):
     *   a_i = G sum_j m_j (x_j - x_i) / (|x_j - x_i|^2 + eps2)^{3/2}
     *   v_i += a_i dt;  x_i += v_i dt      for targets i in [0, n_tgt)
     * args: pos_src:R f32x4[n_src] (x, y, z, m of ALL bodies),
     *       vel:RW f32x4[n_tgt] (vx, vy, vz, 0 of the targets),
     *       pos_out:W f32x4[n_tgt] (x, y, z, m of the targets after the step);
     * target i is body tgt_offset + i of pos_src.  params jacc_nbody_params_t
     * (eps2 > 0).  n_src <= 65535 * 2048 per task (JACC_ERR_UNSUPPORTED
     * beyond: shard the sources' chunks over tasks/ranks).                 */
    JACC_OP_NBODY_STEP_F32 = 7,
    /* Collectives over the graph's NCCL communicator (north_star; SPMD, one
     * process per GPU, reading R17).  world == 1 without a communicator is
     * the identity (allreduce, broadcast) or a device copy (allgather).
     *   ALLREDUCE_SUM: buf:RW {i32|f32}[n]
     *   ALLGATHER:     send:R {i32|f32|f32x4}[n], recv:W same dtype [n*world]
     *   BROADCAST:     buf:RW [n]; params jacc_bcast_params_t              */
    JACC_OP_ALLREDUCE_SUM = 8,
    JACC_OP_ALLGATHER = 9,
    JACC_OP_BROADCAST = 10,
    /* 2D convolution ("convolves a 2048 x 2048
     * image with a 5 x 5 filter"; reading R20): true convolution, zero
     * padding, same-size output,
     *   out[y][x] = sum_{i,j} f[i][j] img[y + r - i][x + r - j].
     * args: img:R f32[H*W] (row-major), filter:R f32[(2r+1)^2],
     * out:W f32[H*W]; params jacc_conv2d_params_t (1 <= r <= 4).
     * flags JACC_CONV2D_HALO_ROWS: img is a row band WITH its halos,
     * f32[(H+2r)*W] = [r rows above][H rows][r rows below] (what
     * JACC_OP_HALO_EXCHANGE_F32 writes), out f32[H*W] is the band's rows of
     * the whole image's convolution (zero padding in x only).              */
    JACC_OP_CONV2D_F32 = 11,
    /* Correlation matrix (P:494 OpenBitSet "intersection
     * count", P:602 `popc`; reading R21):
     *   C[i][j] = sum_w popcount(A_i[w] & B_j[w]).
     * args: A:R i32[ta*words] (term bitsets, bit d%32 of word d/32 =
     * document d), B:R i32[tb*words] (may be the same buffer as A),
     * C:W i32[ta*tb]; params jacc_corr_params_t.  Bit-exact.                */
    JACC_OP_CORR_POPC_U32 = 12,
    /* Sparse matrix-vector product, CSR (R22):
     *   y[i] = sum_{k=row_ptr[i]}^{row_ptr[i+1]-1} val[k] x[col[k]].
     * args: row_ptr:R i32[n+1], col:R i32[nnz], val:R f32[nnz],
     * x:R f32[ncols], y:W f32[n]; params jacc_spmv_params_t.  The caller
     * guarantees 0 <= row_ptr[i] <= row_ptr[i+1] <= nnz, 0 <= col < ncols. */
    JACC_OP_SPMV_CSR_F32 = 13,
    /* Halo exchange of an image split into row bands over the ranks (SURVEY
     * §8(f) f1: 2D convolution "shards by row bands with a 2-row halo
     * exchange").  Collective (SPMD): rank q's band is rows
     * [lo_q, lo_q + rows) of one image, the bands of ranks 0 .. world-1
     * consecutive and in rank order.
     *   band:R f32[rows*W], ext:W f32[(rows+2r)*W]; params jacc_halo_params_t
     * ext = [r rows above the band: the last r rows of rank q-1's band, zeros
     * on rank 0][band][r rows below: the first r rows of rank q+1's band,
     * zeros on the last rank].  rows >= r on every rank (else
     * JACC_ERR_UNSUPPORTED on that rank).  Peer-memory form under
     * JACC_GRAPH_P2P, ncclSend/ncclRecv otherwise, a local copy at world 1. */
    JACC_OP_HALO_EXCHANGE_F32 = 14
} jacc_op_t;

typedef struct jacc_halo_params {
    int64_t rows, W;        /* this rank's band rows, image columns            */
    int32_t radius;         /* halo rows on each side (the filter radius)      */
    int32_t reserved;
} jacc_halo_params_t;

#define JACC_CONV2D_HALO_ROWS 1u   /* jacc_conv2d_params_t.flags */

typedef struct jacc_corr_params {
    int64_t ta, tb, words;  /* terms of A, terms of B, 32-bit words per term   */
} jacc_corr_params_t;

typedef struct jacc_spmv_params {
    int64_t n, ncols;       /* rows, columns                                  */
} jacc_spmv_params_t;

typedef struct jacc_conv2d_params {
    int64_t H, W;       /* image rows, columns                                 */
    int32_t radius;     /* filter is (2 radius + 1)^2, radius in [1, 4]        */
    uint32_t flags;     /* 0 or JACC_CONV2D_HALO_ROWS                          */
} jacc_conv2d_params_t;

typedef struct jacc_hist_params {
    int32_t nbins;      /* 1 .. 4096 (the sm_100a fast path is nbins <= 256) */
} jacc_hist_params_t;

#define JACC_SGEMM_3XTF32 0 /* tcgen05 kind::tf32, A.B ~ Ah.Bh + Ah.Bl + Al.Bh */
#define JACC_SGEMM_FFMA 1   /* plain fp32 FFMA SIMT kernel (parity baseline)   */
typedef struct jacc_sgemm_params {
    int64_t M, N, K;    /* C is M x N, A is M x K, B is K x N                */
    int64_t lda, ldb, ldc; /* row strides in elements (>= K, N, N)          */
    int32_t mode;       /* JACC_SGEMM_3XTF32 | JACC_SGEMM_FFMA              */
    int32_t reserved;
} jacc_sgemm_params_t;

typedef struct jacc_nbody_params {
    int64_t tgt_offset; /* index in pos_src of target 0                    */
    float dt, eps2, G;  /* eps2 > 0 required (the self term is then 0)     */
    float reserved;
} jacc_nbody_params_t;

typedef struct jacc_bcast_params {
    int32_t root;
} jacc_bcast_params_t;

/* One task argument.  `ptr` is a HOST pointer (the runtime owns a device
 * copy and transfers it as the plan requires) unless flags has
 * JACC_ARG_DEVICE.  Host buffers are identified by their exact byte range
 * [ptr, ptr + count * sizeof(dtype)); two arguments naming the same range
 * are the same buffer; a partial overlap is JACC_ERR_ALIAS.  Host memory
 * stays caller-owned; pinned memory is strongly recommended (pageable
 * memory works but cannot overlap copies with compute).                 */
typedef struct jacc_arg {
    void *ptr;
    uint64_t count;     /* elements of dtype */
    int32_t dtype;      /* jacc_dtype_t */
    uint32_t access;    /* JACC_READ | JACC_WRITE | JACC_READWRITE */
    uint32_t flags;     /* JACC_ARG_DEVICE | JACC_ARG_CACHABLE */
    uint32_t reserved;
} jacc_arg_t;

/* Launch schedule ("lines 6-7 ... defining how the
 * iteration space is mapped onto individual threads" / thread groups of
 * BLOCK_SIZE).  Advisory (R15): every kernel is grid-stride or tiled, so
 * any schedule gives the same result; 0 fields mean "auto" (a multiple of
 * the 148 SMs).  global[0] = total threads, group[0] = threads per group. */
typedef struct jacc_schedule {
    int64_t global[3];
    int32_t group[3];
    int32_t reserved;
} jacc_schedule_t;

/* Device memory allocator hooks (PyTorch's caching allocator in the
 * Python binding).  NULL -> cudaMalloc/cudaFree.                         */
typedef void *(*jacc_alloc_fn)(size_t bytes, int device, void *stream, void *ctx);
typedef void (*jacc_free_fn)(void *ptr, size_t bytes, int device, void *stream, void *ctx);

typedef struct jacc_config {
    int32_t device;     /* CUDA ordinal the graph's tasks run on           */
    int32_t rank;       /* SPMD rank (0 when world == 1)                   */
    int32_t world;      /* number of ranks sharing nccl_comm (>= 1)        */
    uint32_t flags;     /* JACC_GRAPH_*                                     */
    void *nccl_comm;    /* ncclComm_t (e.g. from torch ProcessGroupNCCL
                           _comm_ptr()), or NULL if world == 1             */
    int32_t n_compute;  /* 0..JACC_MAX_STREAMS compute streams given below;
                           0 -> the runtime creates 4 non-blocking streams  */
    int32_t fail_task;  /* test hook: 0 = off; k > 0 makes issuing task k-1
                           fail with JACC_ERR_INJECTED (before its kernel) */
    void *compute[JACC_MAX_STREAMS]; /* cudaStream_t handles (borrowed)    */
    void *h2d;          /* cudaStream_t for host->device copies, or NULL   */
    void *d2h;          /* cudaStream_t for device->host copies, or NULL   */
    void *comm;         /* cudaStream_t for collectives, or NULL           */
    jacc_alloc_fn alloc;
    jacc_free_fn free;
    void *alloc_ctx;
} jacc_config_t;

typedef struct jacc_graph jacc_graph_t;

/* Exported description of one rank's peer window (JACC_GRAPH_P2P): a CUDA
 * IPC memory handle plus its size.  Opaque bytes for the caller, who moves
 * them between ranks (e.g. torch.distributed.all_gather_object).           */
typedef struct jacc_peer_handle {
    unsigned char ipc[64];  /* cudaIpcMemHandle_t of the window base          */
    uint64_t window_bytes;  /* identical on every rank                        */
    int32_t rank;           /* the exporting rank                             */
    int32_t device;         /* its CUDA ordinal (diagnostics only)            */
} jacc_peer_handle_t;

/* Counters of the LAST execute (as planned and issued), then cumulative
 * totals since create.  Verified against the oracle's transfer model in
 * the counted-copies tests.                             */
typedef struct jacc_stats {
    uint64_t h2d_count, h2d_bytes, d2h_count, d2h_bytes;
    uint64_t memsets, kernels, collectives, launches; /* launches = CUDA
                           kernels launched (an op may launch > 1)        */
    uint64_t total_h2d_count, total_h2d_bytes, total_d2h_count, total_d2h_bytes;
    uint64_t total_kernels, total_collectives, total_launches, executes;
    int32_t n_tasks, n_buffers;
    int32_t state;      /* 0 BUILDING, 1 EXECUTING, 2 DONE, 3 FAILED       */
    int32_t reserved;
    uint64_t graph_captures, graph_replays; /* JACC_GRAPH_REPLAY counters   */
} jacc_stats_t;

/* ------------------------------------------------------------ entry points */

/* Create an empty graph (state BUILDING).  cfg is copied; the streams,
 * communicator and allocator it names are borrowed and must outlive the
 * graph.  No CUDA call is made here: resources are acquired at the first
 * execute, so graphs can be built, planned and dumped without a GPU.
 * Errors: JACC_ERR_INVALID_ARG (NULL, world < 1, rank out of range,
 * n_compute out of range, world > 1 without nccl_comm).                  */
int jacc_graph_create(jacc_graph_t **g, const jacc_config_t *cfg);

/* Append a task (ids 0, 1, ... in insertion order) and infer its edges to
 * every earlier task (RAW, WAR, WAW on a common buffer; none for
 * read-read, reading R9).  params: the op's parameter struct (NULL/0 for
 * ops without one); sched: NULL = auto; device: must equal cfg->device
 * (one process per GPU).  Allowed unless EXECUTING; the plan is rebuilt at
 * the next execute.  Errors: _STATE, _INVALID_ARG (count/dtype/params),
 * _ACCESS, _ALIAS, _DEVICE, _UNSUPPORTED.                                */
int jacc_graph_add_task(jacc_graph_t *g, jacc_op_t op, const jacc_arg_t *args, int nargs,
                        const void *params, size_t params_size, const jacc_schedule_t *sched,
                        int device, int *task_id);

/* Plan (if needed) and issue every action asynchronously, then return:
 * H2D copies on the h2d stream, kernels on compute streams waiting only on
 * the events of their own inputs and predecessors (out-of-order issue of
 * independent tasks, R6), collectives on the comm stream, one D2H per
 * host-stale buffer after its last writer.  State -> EXECUTING.  Errors:
 * _STATE (already EXECUTING), _OOM, _CUDA, _NCCL, _INJECTED (state ->
 * FAILED; no D2H was issued, host buffers are untouched, R8).            */
int jacc_graph_execute(jacc_graph_t *g);

/* Block until every action of the current execute has finished.  On
 * success every WRITE/READWRITE host buffer holds its final value and the
 * state is DONE; otherwise FAILED with the first error kept.             */
int jacc_graph_sync(jacc_graph_t *g);

/* Counters; callable in any state. */
int jacc_graph_stats(const jacc_graph_t *g, jacc_stats_t *out);

/* Device milliseconds of task `task_id` in the last completed execute
 * (CUDA events recorded on the stream the task's kernels ran on).
 * Errors: _NOT_FOUND, _STATE (no completed execute).                     */
int jacc_graph_task_ms(const jacc_graph_t *g, int task_id, float *ms);

/* Test hook: change the graph's jacc_config_t.fail_task between executes
 * (0 = off; k > 0 makes issuing task k-1 fail with JACC_ERR_INJECTED), so a
 * test can fail one execute and then run the same graph again (R8: a failed
 * execute leaves host buffers untouched and drops every device residency).
 * Errors: _INVALID_ARG (k < 0), _STATE (EXECUTING).                      */
int jacc_graph_set_fail_task(jacc_graph_t *g, int32_t fail_task);

/* Plan (without executing) and write a stable text dump of the edges and
 * the lowered action list (golden tests; cf. SPEC --dump-actions S:460).
 * Writes at most cap bytes (NUL-terminated); *needed = full size + 1.
 * buf may be NULL to query the size.  Errors: _INVALID_ARG.              */
int jacc_graph_dump(jacc_graph_t *g, char *buf, size_t cap, size_t *needed);

/* The host modified a (CACHABLE) buffer between executes: the next execute
 * copies it in again (reading R5).  Errors: _NOT_FOUND, _STATE.          */
int jacc_buffer_invalidate(jacc_graph_t *g, const void *host_ptr);

/* Implicit sync, then release the device copies, events and owned streams.
 * A connected JACC_GRAPH_P2P graph first waits (on the device) until every
 * rank has reached its destroy, so no peer stores into a freed window:
 * every rank must destroy its graph (SPMD).                              */
int jacc_graph_destroy(jacc_graph_t *g);

/* ---- peer windows (JACC_GRAPH_P2P, reading R23) -------------------------
 * Sequence on every rank: create (flags | JACC_GRAPH_P2P) -> jacc_peer_init
 * -> exchange the handles -> jacc_peer_connect -> jacc_peer_alloc / add_task
 * (same order on every rank) -> execute ...  A world-1 graph needs neither
 * init nor connect (the first execute creates a local window).
 *
 * jacc_peer_init: cudaMalloc a zeroed window of window_bytes (0 -> 64 MiB;
 * at least the 256 KiB flag header) on the graph's device and return its
 * handle.  Errors: _STATE (not a P2P graph, or already initialised), _OOM,
 * _CUDA.                                                                   */
int jacc_peer_init(jacc_graph_t *g, size_t window_bytes, jacc_peer_handle_t *out);

/* Map the other ranks' windows.  handles[q] is rank q's handle, n == world;
 * handles[rank] must be this graph's own.  Errors: _STATE (no init, or
 * already connected), _INVALID_ARG (n, rank order, window sizes differ),
 * _CUDA (cudaIpcOpenMemHandle: the GPUs cannot reach each other).          */
int jacc_peer_connect(jacc_graph_t *g, const jacc_peer_handle_t *handles, int n);

/* Allocate `bytes` (256-byte aligned) of the window for the caller: a
 * device buffer at the SAME offset on every rank, so peers can store into
 * it.  A DEVICE argument that a P2P collective writes from other ranks (the
 * receive buffer of an ALLGATHER, the buffer of a BROADCAST) must come from
 * here.  Owned by the graph (freed by destroy).  Errors: _STATE (no window),
 * _OOM (window full).                                                      */
int jacc_peer_alloc(jacc_graph_t *g, size_t bytes, void **dptr);

const char *jacc_status_string(int status);
const char *jacc_last_error(void);   /* thread-local detail of the last error */
int jacc_abi_version(void);
/* sizeof of an ABI struct by name ("jacc_arg_t", "jacc_config_t", ...), 0 if
 * unknown: lets bindings check their struct layouts against the library. */
size_t jacc_abi_sizeof(const char *type_name);

#ifdef __cplusplus
}
#endif
#endif /* JACC_H_ */
