"""PyTorch as plumbing for libjacc.so: device memory (caching allocator),
streams and the NCCL communicator of a ProcessGroupNCCL.  No compute here."""
from __future__ import annotations

import torch


def torch_allocator():
    """(alloc, free) hooks for jacc_config_t backed by torch's caching allocator."""
    def alloc(size, device, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(size), int(device), int(stream or 0))
        except Exception:
            return None

    def free(ptr, size, device, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    return alloc, free


def nccl_comm_ptr(group=None) -> int:
    """ncclComm_t of torch's ProcessGroupNCCL (eagerly initialised)."""
    import torch.distributed as dist
    pg = group or dist.group.WORLD
    backend = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
    return int(backend._comm_ptr())


def make_graph(device: int = 0, n_streams: int = 4, rank: int = 0, world: int = 1, nccl_comm: int = 0,
               flags: int = 0, fail_task: int = 0):
    """A jacc Graph on `device` with torch-owned streams and allocator.

    Returns (graph, streams) where streams = dict of torch.cuda.Stream objects
    (compute list, h2d, d2h, comm) that must outlive the graph.
    """
    from .jacc import Graph
    dev = torch.device("cuda", device)
    comp = [torch.cuda.Stream(dev) for _ in range(n_streams)]
    h2d, d2h, comm = torch.cuda.Stream(dev), torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    g = Graph(device=device, rank=rank, world=world, flags=flags, nccl_comm=nccl_comm,
              streams=[s.cuda_stream for s in comp], h2d=h2d.cuda_stream, d2h=d2h.cuda_stream,
              comm=comm.cuda_stream, allocator=torch_allocator(), fail_task=fail_task)
    g._streams_keep = (comp, h2d, d2h, comm)
    return g, {"compute": comp, "h2d": h2d, "d2h": d2h, "comm": comm}


def peer_setup(g, window_bytes: int = 0, group=None) -> None:
    """JACC_GRAPH_P2P plumbing: export this rank's window handle, all-gather
    the handles over torch.distributed (any backend) and map the peers'."""
    import torch.distributed as dist
    from .jacc import jacc_peer_handle_t
    h = g.peer_init(window_bytes)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        g.peer_connect([h])
        return
    raw = bytes(h)
    allh = [None] * world
    dist.all_gather_object(allh, raw, group=group)
    g.peer_connect([jacc_peer_handle_t.from_buffer_copy(b) for b in allh])


class _DevPtr:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


def peer_tensor(g, shape, dtype=torch.float32):
    """A CUDA tensor on window memory from jacc_peer_alloc (zero-copy view,
    owned by the graph: keep the graph alive while the tensor is used)."""
    import math
    esz = torch.empty((), dtype=dtype).element_size()
    n = math.prod(shape)
    ptr = g.peer_alloc(max(1, n) * esz)
    typestr = {torch.float32: "<f4", torch.int32: "<i4"}[dtype]
    return torch.as_tensor(_DevPtr(ptr, shape, typestr), device=torch.device("cuda", g.device))
