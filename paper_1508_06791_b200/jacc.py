"""Thin ctypes binding of libjacc.so (include/jacc.h) -- argument marshalling only.

Every step of the hot path runs in libjacc.so's sm_100a kernels; this module
only mirrors the C structs, loads the library and forwards calls under the
same names (``jacc_graph_create``, ``jacc_graph_add_task``,
``jacc_graph_execute``, ``jacc_graph_sync``, ...).  There is no fallback: if
libjacc.so is missing, importing this module raises.

:class:`Graph` is a convenience wrapper over the same calls that keeps the
Python objects backing the bound buffers alive for the graph's lifetime.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libjacc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1508_06791_b200/build.py` "
                      "(there is no CPU or Python fallback)")
_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------ constants
JACC_OK, JACC_ERR_INVALID_ARG, JACC_ERR_STATE, JACC_ERR_ACCESS, JACC_ERR_ALIAS, JACC_ERR_DEVICE, \
    JACC_ERR_OOM, JACC_ERR_CUDA, JACC_ERR_NCCL, JACC_ERR_NOT_FOUND, JACC_ERR_UNSUPPORTED, \
    JACC_ERR_INJECTED = range(12)
JACC_F32, JACC_I32, JACC_F32X4 = 1, 2, 3
JACC_READ, JACC_WRITE, JACC_READWRITE = 1, 2, 3
JACC_ARG_DEVICE, JACC_ARG_CACHABLE = 1, 2
JACC_GRAPH_NAIVE, JACC_GRAPH_SERIAL, JACC_GRAPH_REPLAY, JACC_GRAPH_MERGE, JACC_GRAPH_P2P = 1, 2, 4, 8, 16
JACC_GRAPH_NO_TIMING = 32
JACC_MAX_STREAMS = 8
JACC_PEER_MAX = 8
JACC_ABI_VERSION = 2
(JACC_OP_VADD_F32, JACC_OP_REDUCE_SUM_F32, JACC_OP_HISTOGRAM_I32, JACC_OP_BLACKSCHOLES_F32,
 JACC_OP_BLACKSCHOLES_SOA_F32, JACC_OP_SGEMM_F32, JACC_OP_NBODY_STEP_F32, JACC_OP_ALLREDUCE_SUM,
 JACC_OP_ALLGATHER, JACC_OP_BROADCAST, JACC_OP_CONV2D_F32, JACC_OP_CORR_POPC_U32,
 JACC_OP_SPMV_CSR_F32, JACC_OP_HALO_EXCHANGE_F32) = range(1, 15)
JACC_CONV2D_HALO_ROWS = 1
JACC_SGEMM_3XTF32, JACC_SGEMM_FFMA = 0, 1
STATE_NAMES = {0: "BUILDING", 1: "EXECUTING", 2: "DONE", 3: "FAILED"}
DTYPE_SIZE = {JACC_F32: 4, JACC_I32: 4, JACC_F32X4: 16}


# ---------------------------------------------------------------- structures
class jacc_arg_t(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("count", ctypes.c_uint64), ("dtype", ctypes.c_int32),
                ("access", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class jacc_schedule_t(ctypes.Structure):
    _fields_ = [("global_", ctypes.c_int64 * 3), ("group", ctypes.c_int32 * 3), ("reserved", ctypes.c_int32)]


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)


class jacc_config_t(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("nccl_comm", ctypes.c_void_p), ("n_compute", ctypes.c_int32),
                ("fail_task", ctypes.c_int32), ("compute", ctypes.c_void_p * JACC_MAX_STREAMS),
                ("h2d", ctypes.c_void_p), ("d2h", ctypes.c_void_p), ("comm", ctypes.c_void_p),
                ("alloc", ALLOC_FN), ("free", FREE_FN), ("alloc_ctx", ctypes.c_void_p)]


_U64 = ctypes.c_uint64


class jacc_stats_t(ctypes.Structure):
    _fields_ = [(n, _U64) for n in (
        "h2d_count", "h2d_bytes", "d2h_count", "d2h_bytes", "memsets", "kernels", "collectives", "launches",
        "total_h2d_count", "total_h2d_bytes", "total_d2h_count", "total_d2h_bytes", "total_kernels",
        "total_collectives", "total_launches", "executes")] + \
        [("n_tasks", ctypes.c_int32), ("n_buffers", ctypes.c_int32), ("state", ctypes.c_int32),
         ("reserved", ctypes.c_int32), ("graph_captures", _U64), ("graph_replays", _U64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_ if n != "reserved"}


class jacc_hist_params_t(ctypes.Structure):
    _fields_ = [("nbins", ctypes.c_int32)]


class jacc_sgemm_params_t(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64), ("lda", ctypes.c_int64),
                ("ldb", ctypes.c_int64), ("ldc", ctypes.c_int64), ("mode", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class jacc_nbody_params_t(ctypes.Structure):
    _fields_ = [("tgt_offset", ctypes.c_int64), ("dt", ctypes.c_float), ("eps2", ctypes.c_float),
                ("G", ctypes.c_float), ("reserved", ctypes.c_float)]


class jacc_bcast_params_t(ctypes.Structure):
    _fields_ = [("root", ctypes.c_int32)]


class jacc_conv2d_params_t(ctypes.Structure):
    _fields_ = [("H", ctypes.c_int64), ("W", ctypes.c_int64), ("radius", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class jacc_halo_params_t(ctypes.Structure):
    _fields_ = [("rows", ctypes.c_int64), ("W", ctypes.c_int64), ("radius", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class jacc_corr_params_t(ctypes.Structure):
    _fields_ = [("ta", ctypes.c_int64), ("tb", ctypes.c_int64), ("words", ctypes.c_int64)]


class jacc_spmv_params_t(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("ncols", ctypes.c_int64)]


class jacc_peer_handle_t(ctypes.Structure):
    _fields_ = [("ipc", ctypes.c_ubyte * 64), ("window_bytes", ctypes.c_uint64), ("rank", ctypes.c_int32),
                ("device", ctypes.c_int32)]


STRUCTS = {"jacc_peer_handle_t": jacc_peer_handle_t, "jacc_corr_params_t": jacc_corr_params_t, "jacc_spmv_params_t": jacc_spmv_params_t,
           "jacc_arg_t": jacc_arg_t, "jacc_schedule_t": jacc_schedule_t, "jacc_config_t": jacc_config_t,
           "jacc_stats_t": jacc_stats_t, "jacc_hist_params_t": jacc_hist_params_t,
           "jacc_sgemm_params_t": jacc_sgemm_params_t, "jacc_nbody_params_t": jacc_nbody_params_t,
           "jacc_bcast_params_t": jacc_bcast_params_t, "jacc_conv2d_params_t": jacc_conv2d_params_t,
           "jacc_halo_params_t": jacc_halo_params_t}

# ------------------------------------------------------------- entry points
_vp = ctypes.c_void_p
_lib.jacc_graph_create.argtypes = [ctypes.POINTER(_vp), ctypes.POINTER(jacc_config_t)]
_lib.jacc_graph_add_task.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(jacc_arg_t), ctypes.c_int, _vp,
                                     ctypes.c_size_t, ctypes.POINTER(jacc_schedule_t), ctypes.c_int,
                                     ctypes.POINTER(ctypes.c_int)]
_lib.jacc_graph_execute.argtypes = [_vp]
_lib.jacc_graph_sync.argtypes = [_vp]
_lib.jacc_graph_stats.argtypes = [_vp, ctypes.POINTER(jacc_stats_t)]
_lib.jacc_graph_task_ms.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
_lib.jacc_graph_set_fail_task.argtypes = [_vp, ctypes.c_int32]
_lib.jacc_graph_dump.argtypes = [_vp, ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
_lib.jacc_buffer_invalidate.argtypes = [_vp, _vp]
_lib.jacc_graph_destroy.argtypes = [_vp]
_lib.jacc_status_string.argtypes = [ctypes.c_int]
_lib.jacc_status_string.restype = ctypes.c_char_p
_lib.jacc_last_error.restype = ctypes.c_char_p
_lib.jacc_abi_sizeof.argtypes = [ctypes.c_char_p]
_lib.jacc_abi_sizeof.restype = ctypes.c_size_t
_lib.jacc_peer_init.argtypes = [_vp, ctypes.c_size_t, ctypes.POINTER(jacc_peer_handle_t)]
_lib.jacc_peer_connect.argtypes = [_vp, ctypes.POINTER(jacc_peer_handle_t), ctypes.c_int]
_lib.jacc_peer_alloc.argtypes = [_vp, ctypes.c_size_t, ctypes.POINTER(_vp)]

EXPORTS = ["jacc_graph_create", "jacc_graph_add_task", "jacc_graph_execute", "jacc_graph_sync",
           "jacc_graph_stats", "jacc_graph_task_ms", "jacc_graph_dump", "jacc_buffer_invalidate",
           "jacc_graph_destroy", "jacc_status_string", "jacc_last_error", "jacc_abi_version",
           "jacc_abi_sizeof", "jacc_peer_init", "jacc_peer_connect", "jacc_peer_alloc",
           "jacc_graph_set_fail_task"]

jacc_graph_create = _lib.jacc_graph_create
jacc_graph_add_task = _lib.jacc_graph_add_task
jacc_graph_execute = _lib.jacc_graph_execute
jacc_graph_sync = _lib.jacc_graph_sync
jacc_graph_stats = _lib.jacc_graph_stats
jacc_graph_task_ms = _lib.jacc_graph_task_ms
jacc_graph_dump = _lib.jacc_graph_dump
jacc_graph_set_fail_task = _lib.jacc_graph_set_fail_task
jacc_buffer_invalidate = _lib.jacc_buffer_invalidate
jacc_graph_destroy = _lib.jacc_graph_destroy
jacc_status_string = _lib.jacc_status_string
jacc_last_error = _lib.jacc_last_error
jacc_abi_version = _lib.jacc_abi_version
jacc_abi_sizeof = _lib.jacc_abi_sizeof
jacc_peer_init = _lib.jacc_peer_init
jacc_peer_connect = _lib.jacc_peer_connect
jacc_peer_alloc = _lib.jacc_peer_alloc

if jacc_abi_version() != JACC_ABI_VERSION:
    raise ImportError(f"{LIB_PATH}: ABI version {jacc_abi_version()} != binding's {JACC_ABI_VERSION} (rebuild)")


class JaccError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        detail = _lib.jacc_last_error().decode(errors="replace")
        super().__init__(f"{where}: {jacc_status_string(status).decode()} ({detail})")


def check(status: int, where: str) -> None:
    if status != JACC_OK:
        raise JaccError(status, where)


# --------------------------------------------------------------- arguments
def arg(ptr: int, count: int, dtype: int, access: int, flags: int = 0) -> jacc_arg_t:
    return jacc_arg_t(ctypes.c_void_p(int(ptr)), int(count), int(dtype), int(access), int(flags), 0)


def _np_dtype(a: np.ndarray, f32x4: bool) -> tuple:
    if a.dtype == np.float32:
        if f32x4:
            if a.size % 4:
                raise ValueError(f"f32x4 buffer of {a.size} floats is not a whole number of float4s")
            return JACC_F32X4, a.size // 4
        return JACC_F32, a.size
    if a.dtype == np.int32:
        return JACC_I32, a.size
    raise TypeError(f"unsupported dtype {a.dtype}")


class Graph:
    """One task graph (include/jacc.h) on one device.

    Buffers are given as numpy arrays (host, transferred by the runtime) or
    torch tensors (CUDA tensors become JACC_ARG_DEVICE args, CPU tensors are
    host buffers).  The objects are kept alive while the graph exists.
    """

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, flags: int = 0, nccl_comm: int = 0,
                 streams=(), h2d: int = 0, d2h: int = 0, comm: int = 0, allocator=None, fail_task: int = 0):
        cfg = jacc_config_t()
        cfg.device, cfg.rank, cfg.world, cfg.flags = device, rank, world, flags
        cfg.nccl_comm = nccl_comm or None
        cfg.n_compute = len(streams)
        cfg.fail_task = fail_task
        for i, s in enumerate(streams):
            cfg.compute[i] = int(s)
        cfg.h2d, cfg.d2h, cfg.comm = (h2d or None), (d2h or None), (comm or None)
        self._alloc_keep = None
        if allocator is not None:
            a, f = allocator
            self._alloc_keep = (ALLOC_FN(a), FREE_FN(f))
            cfg.alloc, cfg.free = self._alloc_keep
        self._cfg = cfg
        self._h = ctypes.c_void_p()
        check(jacc_graph_create(ctypes.byref(self._h), ctypes.byref(cfg)), "jacc_graph_create")
        self.device = device
        self._keep = []

    # -- argument helpers ------------------------------------------------
    def a(self, obj, access: int, cachable: bool = False, f32x4: bool = False) -> jacc_arg_t:
        flags = JACC_ARG_CACHABLE if cachable else 0
        if isinstance(obj, np.ndarray):
            if not obj.flags.c_contiguous:
                raise ValueError("buffer must be C-contiguous")
            dt, n = _np_dtype(obj, f32x4)
            self._keep.append(obj)
            return arg(obj.ctypes.data, n, dt, access, flags)
        import torch  # torch tensors: device memory / pinned host memory
        if isinstance(obj, torch.Tensor):
            if not obj.is_contiguous():
                raise ValueError("tensor must be contiguous")
            dts = {torch.float32: JACC_F32, torch.int32: JACC_I32}
            if obj.dtype not in dts:
                raise TypeError(f"unsupported dtype {obj.dtype}")
            dt = dts[obj.dtype]
            n = obj.numel()
            if f32x4:
                if obj.dtype != torch.float32 or n % 4:
                    raise ValueError(f"f32x4 tensor of {n} {obj.dtype} is not a whole number of float4s")
                dt, n = JACC_F32X4, n // 4
            if obj.is_cuda:
                flags |= JACC_ARG_DEVICE
            self._keep.append(obj)
            return arg(obj.data_ptr(), n, dt, access, flags)
        raise TypeError(type(obj))

    def add_task(self, op: int, args, params=None, sched=None) -> int:
        arr = (jacc_arg_t * len(args))(*args)
        tid = ctypes.c_int(-1)
        pp = ctypes.byref(params) if params is not None else None
        psz = ctypes.sizeof(params) if params is not None else 0
        sp = ctypes.byref(sched) if sched is not None else None
        if params is not None:
            self._keep.append(params)
        check(jacc_graph_add_task(self._h, op, arr, len(args), pp, psz, sp, self.device, ctypes.byref(tid)),
              "jacc_graph_add_task")
        return tid.value

    def execute(self) -> None:
        check(jacc_graph_execute(self._h), "jacc_graph_execute")

    def sync(self) -> None:
        check(jacc_graph_sync(self._h), "jacc_graph_sync")

    def run(self) -> None:
        """The paper's blocking TaskGraph.execute = execute + sync."""
        self.execute()
        self.sync()

    def stats(self) -> dict:
        s = jacc_stats_t()
        check(jacc_graph_stats(self._h, ctypes.byref(s)), "jacc_graph_stats")
        return s.as_dict()

    def task_ms(self, task_id: int) -> float:
        ms = ctypes.c_float()
        check(jacc_graph_task_ms(self._h, task_id, ctypes.byref(ms)), "jacc_graph_task_ms")
        return ms.value

    def set_fail_task(self, fail_task: int) -> None:
        """Test hook (include/jacc.h jacc_graph_set_fail_task)."""
        check(jacc_graph_set_fail_task(self._h, int(fail_task)), "jacc_graph_set_fail_task")

    def dump(self) -> str:
        need = ctypes.c_size_t()
        check(jacc_graph_dump(self._h, None, 0, ctypes.byref(need)), "jacc_graph_dump")
        buf = ctypes.create_string_buffer(need.value)
        check(jacc_graph_dump(self._h, buf, need.value, ctypes.byref(need)), "jacc_graph_dump")
        return buf.value.decode()

    # -- JACC_GRAPH_P2P peer windows (jacc_peer_init / _connect / _alloc) ----
    def peer_init(self, window_bytes: int = 0) -> jacc_peer_handle_t:
        h = jacc_peer_handle_t()
        check(jacc_peer_init(self._h, int(window_bytes), ctypes.byref(h)), "jacc_peer_init")
        return h

    def peer_connect(self, handles) -> None:
        arr = (jacc_peer_handle_t * len(handles))(*handles)
        check(jacc_peer_connect(self._h, arr, len(handles)), "jacc_peer_connect")

    def peer_alloc(self, nbytes: int) -> int:
        """Device pointer of `nbytes` in the symmetric window (same offset on every rank)."""
        p = ctypes.c_void_p()
        check(jacc_peer_alloc(self._h, int(nbytes), ctypes.byref(p)), "jacc_peer_alloc")
        return int(p.value)

    def invalidate(self, obj) -> None:
        ptr = obj.ctypes.data if isinstance(obj, np.ndarray) else obj.data_ptr()
        check(jacc_buffer_invalidate(self._h, ctypes.c_void_p(ptr)), "jacc_buffer_invalidate")

    def destroy(self) -> None:
        if self._h:
            check(jacc_graph_destroy(self._h), "jacc_graph_destroy")
            self._h = ctypes.c_void_p()
            self._keep.clear()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
