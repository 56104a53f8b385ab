"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/jacc.h declares, the binding's struct layouts match the library's,
argument validation, and the runtime's PLANNER (dependency edges, transfer
elision, counted copies, action order) equals the oracle's task-graph model
(oracle/graph_model.py) on the SURVEY count table and on random graphs.
No compute call is made (jacc_graph_create/add_task/dump/stats touch no CUDA).
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
from oracle import graph_model as gm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "jacc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(jacc_\w+)\s*\(", txt)) - {"jacc_alloc_fn", "jacc_free_fn"})


def test_exports_every_declared_symbol():
    declared = _header_functions()
    assert len(declared) >= 12
    out = subprocess.run(["nm", "-D", "--defined-only", J.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (jacc_\w+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    assert sorted(jacc.EXPORTS) == declared
    lib = ctypes.CDLL(J.LIB_PATH)
    for f in declared:
        assert getattr(lib, f)


def test_struct_layouts_match_library():
    for name, S in jacc.STRUCTS.items():
        assert ctypes.sizeof(S) == J.jacc_abi_sizeof(name.encode()), name
    assert J.jacc_abi_sizeof(b"nope") == 0
    assert J.jacc_abi_version() == 2


def test_status_strings():
    assert J.jacc_status_string(0) == b"JACC_OK"
    assert J.jacc_status_string(4) == b"JACC_ERR_ALIAS"


def test_create_validation():
    with pytest.raises(J.JaccError):
        J.Graph(world=2)            # world > 1 needs a communicator
    with pytest.raises(J.JaccError):
        J.Graph(rank=1, world=1)
    g = J.Graph()
    assert g.stats()["state"] == 0
    g.destroy()


def test_add_task_validation():
    g = J.Graph()
    a = np.zeros(16, np.float32); b = np.zeros(16, np.float32); c = np.zeros(16, np.float32)
    with pytest.raises(J.JaccError) as e:   # vadd output must be W
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, 1), g.a(b, 1), g.a(c, 1)])
    assert e.value.status == J.JACC_ERR_ACCESS
    with pytest.raises(J.JaccError) as e:   # count mismatch
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, 1), g.a(b[:8], 1), g.a(c, 2)])
    assert e.value.status == J.JACC_ERR_INVALID_ARG
    with pytest.raises(J.JaccError) as e:   # partial overlap with a registered buffer
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, 1), g.a(b, 1), g.a(c, 2)])
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a[4:12], 1), g.a(b[4:12], 1), g.a(c[:8], 2)])
    assert e.value.status == J.JACC_ERR_ALIAS
    with pytest.raises(J.JaccError) as e:   # written buffer aliasing an input
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, 1), g.a(b, 1), g.a(a, 2)])
    assert e.value.status == J.JACC_ERR_ALIAS
    with pytest.raises(J.JaccError) as e:   # wrong device: one process per GPU
        arr = (jacc.jacc_arg_t * 3)(g.a(a, 1), g.a(b, 1), g.a(c, 2))
        J.check(J.jacc_graph_add_task(g._h, J.JACC_OP_VADD_F32, arr, 3, None, 0, None, 3, None), "x")
    assert e.value.status == J.JACC_ERR_DEVICE
    for bad in (0, 4, 33, 0xFFFFFFFF):      # access outside READ/WRITE/READWRITE
        with pytest.raises(J.JaccError) as e:
            arr = (jacc.jacc_arg_t * 3)(g.a(a, 1), g.a(b, 1), g.a(c, 2))
            arr[2].access = bad
            J.check(J.jacc_graph_add_task(g._h, J.JACC_OP_VADD_F32, arr, 3, None, 0, None, 0, None), "x")
        assert e.value.status == J.JACC_ERR_ACCESS
    img = np.zeros((4, 4), np.float32); f = np.zeros(25, np.float32)
    with pytest.raises(J.JaccError) as e:   # H*W that overflows int32 must not wrap around
        g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img, 1), g.a(f, 1), g.a(np.zeros_like(img), 2)],
                   jacc.jacc_conv2d_params_t(65536, 65536, 2, 0))
    assert e.value.status == J.JACC_ERR_INVALID_ARG
    keys = np.zeros(64, np.int32); bins = np.zeros(300, np.int32)
    with pytest.raises(J.JaccError):        # bins count != nbins
        g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, 1), g.a(bins, 2)], jacc.jacc_hist_params_t(256))
    pos = np.zeros((8, 4), np.float32); vel = np.zeros((8, 4), np.float32); out = np.zeros((8, 4), np.float32)
    with pytest.raises(J.JaccError):        # eps2 must be > 0
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(pos, 1, f32x4=True), g.a(vel, 3, f32x4=True),
                                               g.a(out, 2, f32x4=True)], jacc.jacc_nbody_params_t(0, 0.01, 0.0, 1.0))
    g.destroy()


# ------------------------------------------------ planner == oracle model
class _Pool:
    """Host buffers for random graphs; one fixed dtype/size per name."""

    def __init__(self, n=64):
        self.f = {k: np.zeros(n, np.float32) for k in "ABCDE"}
        self.s = {k: np.zeros(1, np.float32) for k in "st"}
        self.k = {k: np.zeros(n, np.int32) for k in "K"}
        self.h = {k: np.zeros(16, np.int32) for k in "H"}


def _add(g, pool, task):
    """Add a model Task to the C graph with matching ops/buffers."""
    def A(x):
        arr = {**pool.f, **pool.s, **pool.k, **pool.h}[x.buf]
        return g.a(arr, x.access, cachable=x.cachable)
    op = task.op
    if op == "vadd":
        return g.add_task(J.JACC_OP_VADD_F32, [A(x) for x in task.args])
    if op == "reduce":
        return g.add_task(J.JACC_OP_REDUCE_SUM_F32, [A(x) for x in task.args])
    if op == "hist":
        return g.add_task(J.JACC_OP_HISTOGRAM_I32, [A(x) for x in task.args], jacc.jacc_hist_params_t(16))
    if op == "allreduce":
        return g.add_task(J.JACC_OP_ALLREDUCE_SUM, [A(x) for x in task.args])
    if op == "allgather":
        return g.add_task(J.JACC_OP_ALLGATHER, [A(x) for x in task.args])
    raise ValueError(op)


def _random_tasks(rng, ntask):
    R, W, RW = gm.READ, gm.WRITE, gm.READWRITE
    tasks = []
    for _ in range(ntask):
        kind = rng.integers(0, 5)
        f = list("ABCDE")
        if kind == 0:
            i, j, o = rng.choice(f, 3, replace=True)
            if o in (i, j):
                continue
            tasks.append(gm.Task("vadd", [gm.Arg(i, R, cachable=bool(rng.integers(2))),
                                          gm.Arg(j, R), gm.Arg(o, W)]))
        elif kind == 1:
            tasks.append(gm.Task("reduce", [gm.Arg(rng.choice(f), R),
                                            gm.Arg(rng.choice(["s", "t"]), [W, RW][rng.integers(2)])]))
        elif kind == 2:
            tasks.append(gm.Task("hist", [gm.Arg("K", R, cachable=True), gm.Arg("H", [W, RW][rng.integers(2)])]))
        elif kind == 3:
            tasks.append(gm.Task("allreduce", [gm.Arg(rng.choice(f + ["s", "t", "H"]), RW)]))
        else:
            i, o = rng.choice(f, 2, replace=False)
            tasks.append(gm.Task("allgather", [gm.Arg(i, R), gm.Arg(o, W)]))
    return tasks


def _c_actions(dump, names):
    acts = []
    for line in dump.splitlines():
        p = line.split()
        if p[0] != "action":
            continue
        if p[1] in ("H2D", "D2H", "MEMSET0"):
            acts.append((p[1], names[int(p[2][1:])]))
        else:
            acts.append((p[1], int(p[2][1:]), p[3]))
    return acts


def _c_edges(dump):
    return sorted((int(p[1]), int(p[2])) for p in (l.split() for l in dump.splitlines()) if p[0] == "edge")


@pytest.mark.parametrize("naive", [False, True])
def test_planner_equals_model_random(naive):
    rng = np.random.default_rng(123 + naive)
    for trial in range(150):
        pool = _Pool()
        tasks = _random_tasks(rng, int(rng.integers(1, 9)))
        if not tasks:
            continue
        g = J.Graph(flags=J.JACC_GRAPH_NAIVE if naive else 0)
        for t in tasks:
            _add(g, pool, t)
        names = gm.buffer_order(tasks)
        d = g.dump()
        assert _c_actions(d, names) == gm.plan(tasks, naive=naive), (d, tasks)
        assert _c_edges(d) == gm.infer_edges(tasks)
        st = g.stats()
        c = gm.counts(gm.plan(tasks, naive=naive))
        assert (st["h2d_count"], st["d2h_count"], st["memsets"], st["kernels"], st["collectives"]) == \
            (c["H2D"], c["D2H"], c["MEMSET0"], c["KERNEL"], c["COLLECTIVE"])
        g.destroy()


def test_survey_cfg1_counts_and_bytes():
    n = 1 << 20
    a = np.zeros(n, np.float32); b = np.zeros(n, np.float32); c = np.zeros(n, np.float32)
    s = np.zeros(1, np.float32)
    for naive, want in ((True, (3, 2, 3 * 4 * n, 4 * n + 4)), (False, (2, 2, 2 * 4 * n, 4 * n + 4))):
        g = J.Graph(flags=J.JACC_GRAPH_NAIVE if naive else 0)
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, 1, True), g.a(b, 1, True), g.a(c, 2)])
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, 1), g.a(s, 2)])
        st = g.stats()
        assert (st["h2d_count"], st["d2h_count"], st["h2d_bytes"], st["d2h_bytes"]) == want
        g.destroy()


def test_independent_tasks_spread_over_streams():
    # out-of-order issue (R6): independent chains get distinct compute streams
    pool = _Pool()
    g = J.Graph()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(pool.f["A"], 1), g.a(pool.f["B"], 1), g.a(pool.f["C"], 2)])
    g.add_task(J.JACC_OP_VADD_F32, [g.a(pool.f["D"], 1), g.a(pool.f["B"], 1), g.a(pool.f["E"], 2)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(pool.f["C"], 1), g.a(pool.s["s"], 2)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(pool.f["E"], 1), g.a(pool.s["t"], 2)])
    d = g.dump()
    streams = [int(re.search(r"stream=(-?\d+)", l).group(1)) for l in d.splitlines() if l.startswith("task")]
    assert streams[0] != streams[1]
    assert streams[2] == streams[0] and streams[3] == streams[1]
    g.destroy()


def test_p2p_create_and_window_state():
    # JACC_GRAPH_P2P: world > 1 needs no NCCL communicator, but a window
    g = J.Graph(rank=1, world=2, flags=J.JACC_GRAPH_P2P)
    with pytest.raises(J.JaccError, match="STATE"):
        g.peer_alloc(1024)                    # no jacc_peer_init yet
    with pytest.raises(J.JaccError, match="STATE"):
        g.peer_connect([jacc.jacc_peer_handle_t(), jacc.jacc_peer_handle_t()])
    g.destroy()
    with pytest.raises(J.JaccError, match="INVALID_ARG"):
        J.Graph(world=9, flags=J.JACC_GRAPH_P2P)   # one NVLink domain: <= JACC_PEER_MAX ranks
    g = J.Graph(flags=J.JACC_GRAPH_NAIVE)
    with pytest.raises(J.JaccError, match="STATE"):
        g.peer_init(0)                        # not a P2P graph
    g.destroy()


def _p2p_fusions(flags=0, world=2):
    """Fusion lines of the dump of the bench's per-rank graph shape."""
    n = 64
    g = J.Graph(rank=0, world=world, flags=J.JACC_GRAPH_P2P | flags)
    keys = np.zeros(1000, np.int32); bins = np.zeros(256, np.int32)
    x = np.zeros(10, np.float32); s = np.zeros(1, np.float32)
    big = np.zeros(600, np.int32); bins2 = np.zeros(300, np.int32)
    L = [np.zeros((n // world, 4), np.float32) for _ in range(2)]
    V = np.zeros((n // world, 4), np.float32)
    ALL = np.zeros((n, 4), np.float32)
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, 1), g.a(bins, 2)], jacc.jacc_hist_params_t(256))
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(bins, 3)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, 1), g.a(s, 2)])
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(s, 3)])
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, 1), g.a(bins2, 2)], jacc.jacc_hist_params_t(300))
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(bins2, 3)])      # nbins > 256: not fused
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(big, 3)])        # no producer: standalone
    for k in range(3):
        g.add_task(J.JACC_OP_ALLGATHER, [g.a(L[k % 2], 1, f32x4=True), g.a(ALL, 2, f32x4=True)])
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(ALL, 1, f32x4=True), g.a(V, 3, f32x4=True),
                                               g.a(L[(k + 1) % 2], 2, f32x4=True)],
                   jacc.jacc_nbody_params_t(0, 0.016, 0.01, 1.0))
    d = g.dump()
    g.destroy()
    return [l for l in d.splitlines() if l.startswith("fuse")]


def test_p2p_fusion_rule():
    """Reading R23: a collective fused into the kernel that produces its data
    (hist -> allreduce(bins), reduce -> allreduce(out), nbody ->
    allgather(pos_out)); collectives get slots in insertion order."""
    f = _p2p_fusions()
    assert f == ["fuse t0 hist + t1 allreduce slot=0", "fuse t2 reduce + t3 allreduce slot=1",
                 "fuse t8 nbody + t9 allgather slot=5", "fuse t10 nbody + t11 allgather slot=6"], f
    assert _p2p_fusions(J.JACC_GRAPH_NAIVE) == []    # the naive lowering fuses nothing
