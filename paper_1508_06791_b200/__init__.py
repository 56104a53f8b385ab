"""paper_1508_06791_b200 -- B200-native (sm_100a) Jacc task-graph runtime.

The product is the C-ABI library ``libjacc.so`` (include/jacc.h): a task
graph runtime with dependency inference, transfer elision, out-of-order issue
and hand-written sm_100a kernels (vector add, reduction, histogram,
Black-Scholes, SGEMM 3xTF32 on tcgen05, N-body) plus NCCL collectives.
``jacc`` is the thin ctypes binding; ``torch_glue`` lends PyTorch's caching
allocator, streams and NCCL communicator to it (plumbing only).
"""
from .jacc import *  # noqa: F401,F403
from .jacc import Graph, JaccError, LIB_PATH  # noqa: F401

__all__ = [n for n in dir() if n.startswith(("jacc_", "JACC_"))] + ["Graph", "JaccError", "LIB_PATH"]
