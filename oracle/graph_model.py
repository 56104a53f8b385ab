"""Task-graph semantics oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Follows PAPER.md §2 / §2.3 and SURVEY.md §8(c)-G:

* a task is "a method reference, a parameter list and some scheduling
  metadata"; per-parameter access is @Read / @Write / @ReadWrite
  (Table 1);
* "it is possible to infer all the data dependencies between tasks":
  :func:`infer_edges` -- edge i->j (i < j) iff both touch one buffer and at
  least one writes it (RAW, WAR, WAW); read-read gives no edge (R9);
* each task is lowered into "data transfers to the GPU, code execution on
  the GPU, and data transfers back to the host", and the
  runtime eliminates the redundant ones:
  :func:`plan` is the transfer model G.3 (reading R3), with the naive
  lowering as ``naive=True``;
* an @Atomic output written by a task is "automatically initialise[d] to
  zero": MEMSET0 on the device, never a transfer (R10);
* the serial semantics -- "the underlying Java code still produces a correct
  result if it is executed in a serial manner" -- is
  :func:`serial_execute`, the reference every graph result must equal.

Pinned by tests/test_graph_model.py against brute-force minimal copy sets
and the SPEC's worked examples.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

READ, WRITE, READWRITE = 1, 2, 3

# op -> tuple of (access-set allowed per arg, is_atomic_output) ; the model's
# own table of the op signatures (SURVEY §8(b) "Ops").
OPS = {
    "vadd": ((READ,), (READ,), (WRITE,)),
    "reduce": ((READ,), (WRITE, READWRITE)),
    "hist": ((READ,), (WRITE, READWRITE)),
    "bs": ((READ,), (WRITE,), (WRITE,)),
    "bs_soa": ((READ,),) * 5 + ((WRITE,), (WRITE,)),
    "sgemm": ((READ,), (READ,), (WRITE,)),
    "nbody": ((READ,), (READWRITE,), (WRITE,)),
    "allreduce": ((READWRITE,),),
    "allgather": ((READ,), (WRITE,)),
    "broadcast": ((READWRITE,),),
    "conv2d": ((READ,), (READ,), (WRITE,)),
    "corr": ((READ,), (READ,), (WRITE,)),
    "spmv": ((READ,),) * 4 + ((WRITE,),),
    "halo": ((READ,), (WRITE,)),
}
ATOMIC_OUT = {"reduce": 1, "hist": 1}   # arg index of the @Atomic(op=ADD) output
COLLECTIVES = {"allreduce", "allgather", "broadcast", "halo"}


@dataclass
class Arg:
    buf: str          # buffer identity (host range)
    access: int       # READ / WRITE / READWRITE
    device: bool = False     # caller-owned device buffer: never transferred
    cachable: bool = False   # may stay resident across executes (R5)


@dataclass
class Task:
    op: str
    args: list
    params: dict = field(default_factory=dict)


def infer_edges(tasks):
    """Edges (i, j), i < j: common buffer and at least one side writes it."""
    edges = set()
    for j, tj in enumerate(tasks):
        for i in range(j):
            ti = tasks[i]
            for a in ti.args:
                for b in tj.args:
                    if a.buf == b.buf and ((a.access & WRITE) or (b.access & WRITE)):
                        edges.add((i, j))
    return sorted(edges)


def buffer_order(tasks):
    order = []
    for t in tasks:
        for a in t.args:
            if a.buf not in order:
                order.append(a.buf)
    return order


def plan(tasks, resident=None, naive=False):
    """Lowered action list for one execute.

    resident: set of buffer names whose device copy is current at the start
    (CACHABLE, not invalidated, copied in by an earlier execute).
    Returns a list of tuples: ("H2D", buf) | ("MEMSET0", buf) |
    ("KERNEL", i, op) | ("COLLECTIVE", i, op) | ("D2H", buf).
    """
    resident = set(resident or ())
    dev_valid = {}
    host_valid = {}
    last_writer = {}
    is_device = {}
    for b in buffer_order(tasks):
        dev_valid[b] = b in resident
        host_valid[b] = True
    for t in tasks:
        for a in t.args:
            is_device[a.buf] = is_device.get(a.buf, False) or a.device
    actions = []
    for i, t in enumerate(tasks):
        atomic = ATOMIC_OUT.get(t.op)
        for k, a in enumerate(t.args):
            if a.device:
                continue
            if a.access & READ:
                if naive or not dev_valid[a.buf]:
                    actions.append(("H2D", a.buf))
                    dev_valid[a.buf] = True
        for k, a in enumerate(t.args):
            if atomic == k and a.access == WRITE:
                actions.append(("MEMSET0", a.buf))
        actions.append(("COLLECTIVE" if t.op in COLLECTIVES else "KERNEL", i, t.op))
        for k, a in enumerate(t.args):
            if a.access & WRITE:
                dev_valid[a.buf] = True
                host_valid[a.buf] = False
                last_writer[a.buf] = i
                if naive and not a.device:
                    actions.append(("D2H", a.buf))
                    host_valid[a.buf] = True
    if not naive:
        # one D2H per stale host buffer, after its last writer; ordered by
        # (last writer, first appearance) for a stable dump
        order = buffer_order(tasks)
        stale = [b for b in order if not host_valid[b] and not is_device[b]]
        stale.sort(key=lambda b: (last_writer[b], order.index(b)))
        actions.extend(("D2H", b) for b in stale)
    return actions


def counts(actions):
    c = {"H2D": 0, "D2H": 0, "MEMSET0": 0, "KERNEL": 0, "COLLECTIVE": 0}
    for a in actions:
        c[a[0]] += 1
    return c


# ------------------------------------------------------------ serial executor
def serial_execute(tasks, host, kernels):
    """Run tasks one by one in insertion order on copies of the host buffers.

    host: dict buf -> numpy array (not modified).  kernels: dict op ->
    callable(task, arrays) that updates the arrays in place (the oracle's
    kernel functions).  Returns the final host state.
    """
    state = {k: np.array(v, copy=True) for k, v in host.items()}
    for t in tasks:
        arrays = [state[a.buf] for a in t.args]
        atomic = ATOMIC_OUT.get(t.op)
        if atomic is not None and t.args[atomic].access == WRITE:
            arrays[atomic][...] = 0        # auto-zero
        kernels[t.op](t, arrays)
    return state
