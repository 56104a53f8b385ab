"""Pins for the task-graph semantics oracle (oracle/graph_model.py) -- CPU only.

* SPEC worked examples (tests/golden/spec_examples.json);
* the transfer-elision model equals a BRUTE-FORCE minimum: on every graph of
  <= 3 tasks over <= 3 buffers, the smallest subset of the naive copy list
  (plus end-of-graph D2H slots) that keeps every kernel reading the latest
  version of its inputs and leaves the host with the latest version of every
  buffer has exactly the model's H2D and D2H counts;
* the count table of SURVEY §8(c)-G for the BASELINE configs.
"""
import itertools
import json
import os

import pytest

from oracle.graph_model import (ATOMIC_OUT, READ, READWRITE, WRITE, Arg, Task, counts,
                                infer_edges, plan)

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_spec_edges():
    # RAW edge, RR no edge, WAR edge
    assert infer_edges([Task("vadd", [Arg("A", READ), Arg("B", READ), Arg("C", WRITE)]),
                        Task("reduce", [Arg("C", READ), Arg("s", WRITE)])]) == [(0, 1)]
    assert infer_edges([Task("reduce", [Arg("A", READ), Arg("s", WRITE)]),
                        Task("reduce", [Arg("A", READ), Arg("t", WRITE)])]) == []
    assert infer_edges([Task("reduce", [Arg("A", READ), Arg("s", WRITE)]),
                        Task("vadd", [Arg("X", READ), Arg("Y", READ), Arg("A", WRITE)])]) == [(0, 1)]


def test_spec_vadd_naive_lowering():
    g = GOLDEN["vadd_naive_lowering"]
    c = counts(plan([Task("vadd", [Arg("a", READ), Arg("b", READ), Arg("c", WRITE)])], naive=True))
    assert (c["H2D"], c["KERNEL"], c["D2H"]) == (g["copy_in"], g["execute"], g["copy_out"])


def test_spec_chain_elision():
    g = GOLDEN["transfer_chain_elision"]
    tasks = [Task("nbody", [Arg("P", READ), Arg("A", READWRITE), Arg("Q", WRITE)]),
             Task("nbody", [Arg("Q", READ), Arg("A", READWRITE), Arg("P", WRITE)])]
    naive = plan(tasks, naive=True)
    opt = plan(tasks)
    assert sum(1 for a in naive if a == ("H2D", "A")) == g["naive_copy_in_A"]
    assert sum(1 for a in naive if a == ("D2H", "A")) == g["naive_copy_out_A"]
    assert sum(1 for a in opt if a == ("H2D", "A")) == g["optimized_copy_in_A"]
    assert sum(1 for a in opt if a == ("D2H", "A")) == g["optimized_copy_out_A"]


# ------------------------------------------------------------- brute force
def _valid(tasks, chosen, slots, resident):
    """Simulate versions with the chosen copies; True iff every kernel reads
    the latest version and the host ends with the latest of every buffer."""
    bufs = {a.buf for t in tasks for a in t.args}
    latest = {b: 0 for b in bufs}
    host = {b: 0 for b in bufs}
    dev = {b: (0 if b in resident else None) for b in bufs}
    chosen = set(chosen)
    for i, t in enumerate(tasks):
        for s in slots:
            if s[0] == "H2D" and s[1] == i and s in chosen:
                dev[s[2]] = host[s[2]]
        for a in t.args:
            if a.access & READ and dev[a.buf] != latest[a.buf]:
                return False
        for a in t.args:
            if a.access & WRITE:
                latest[a.buf] += 1
                dev[a.buf] = latest[a.buf]
        for s in slots:
            if s[0] == "D2H" and s[1] == i and s in chosen:
                host[s[2]] = dev[s[2]]
    return all(host[b] == latest[b] for b in bufs)


def _brute_min(tasks, resident):
    slots = []
    for i, t in enumerate(tasks):
        for a in t.args:
            if a.access & READ:
                slots.append(("H2D", i, a.buf))
            if a.access & WRITE:
                slots.append(("D2H", i, a.buf))
    slots = sorted(set(slots))
    for k in range(len(slots) + 1):
        for sub in itertools.combinations(slots, k):
            if _valid(tasks, sub, slots, resident):
                return (sum(1 for s in sub if s[0] == "H2D"), sum(1 for s in sub if s[0] == "D2H"))
    raise AssertionError("no valid copy set")


def _graphs():
    # ops with one input and one output arg, or a single RW arg, over 3 buffers
    bufs = "XYZ"
    shapes = []
    for ins in bufs:
        for outs in bufs:
            if ins != outs:
                shapes.append(("red", ins, outs))   # reduce-like: R in, W(atomic) out
                shapes.append(("map", ins, outs))   # map-like: R in, W out
        shapes.append(("rw", ins, None))            # allreduce-like: RW
    for ntask in (1, 2, 3):
        for combo in itertools.product(shapes, repeat=ntask):
            tasks = []
            for kind, i, o in combo:
                if kind == "red":
                    tasks.append(Task("reduce", [Arg(i, READ), Arg(o, WRITE)]))
                elif kind == "map":
                    tasks.append(Task("allgather", [Arg(i, READ), Arg(o, WRITE)]))
                else:
                    tasks.append(Task("allreduce", [Arg(i, READWRITE)]))
            yield tasks


def test_model_equals_brute_force_minimum():
    n = 0
    for tasks in _graphs():
        if n % 3 == 0:   # ~1/3 of the 3-task space keeps the CPU suite fast
            for resident in (set(), {"X"}):
                c = counts(plan(tasks, resident=resident))
                assert (c["H2D"], c["D2H"]) == _brute_min(tasks, resident), tasks
        n += 1
    assert n == 3615


def test_atomic_write_is_memset_not_transfer():
    c = counts(plan([Task("hist", [Arg("k", READ), Arg("bins", WRITE)])]))
    assert (c["H2D"], c["MEMSET0"], c["D2H"]) == (1, 1, 1)
    c = counts(plan([Task("hist", [Arg("k", READ), Arg("bins", READWRITE)])]))
    assert (c["H2D"], c["MEMSET0"], c["D2H"]) == (2, 0, 1)


# ------------------------------------------------ SURVEY §8(c)-G count table
def _cfg1(k=1):
    t = []
    for _ in range(k):
        t.append(Task("vadd", [Arg("a", READ, cachable=True), Arg("b", READ, cachable=True),
                               Arg("c", WRITE)]))
        t.append(Task("reduce", [Arg("c", READ), Arg("s", WRITE)]))
    return t


@pytest.mark.parametrize("name,tasks,naive,elided,second", [
    ("cfg1", _cfg1(), (3, 2), (2, 2), (0, 2)),
    ("cfg1x5", _cfg1(5), (15, 10), (2, 2), (0, 2)),
    ("cfg2", [Task("hist", [Arg("keys", READ, cachable=True), Arg("bins", WRITE)]),
              Task("allreduce", [Arg("bins", READWRITE)])], (2, 2), (1, 1), (0, 1)),
    ("cfg3", [Task("bs", [Arg("u", READ, cachable=True), Arg("call", WRITE), Arg("put", WRITE)])],
     (1, 2), (1, 2), (0, 2)),
    ("cfg4", [Task("sgemm", [Arg("A", READ, cachable=True), Arg("B", READ, cachable=True),
                             Arg("C", WRITE)])], (2, 1), (2, 1), (0, 1)),
    ("cfg5", [Task("nbody", [Arg(f"P{k % 2}", READ, cachable=True), Arg("V", READWRITE, cachable=True),
                             Arg(f"P{(k + 1) % 2}", WRITE, cachable=True)]) for k in range(10)],
     (20, 20), (2, 3), (0, 3)),
    ("cfg5_shard", [t for k in range(10) for t in (
        Task("allgather", [Arg(f"L{k % 2}", READ, cachable=True), Arg("ALL", WRITE, device=True)]),
        Task("nbody", [Arg("ALL", READ, device=True), Arg("V", READWRITE, cachable=True),
                       Arg(f"L{(k + 1) % 2}", WRITE, cachable=True)]))], (20, 20), (2, 3), (0, 3)),
])
def test_survey_count_table(name, tasks, naive, elided, second):
    c = counts(plan(tasks, naive=True))
    assert (c["H2D"], c["D2H"]) == naive
    c = counts(plan(tasks))
    assert (c["H2D"], c["D2H"]) == elided
    resident = {a.buf for t in tasks for a in t.args if a.cachable and not a.device}
    c = counts(plan(tasks, resident=resident))
    assert (c["H2D"], c["D2H"]) == second


# ------------------------------------------------ serial executor
# serial_execute is the reference every GPU graph is compared with
# (tests/test_gpu_graph.py serializability).  Pinned here against final
# states derived BY HAND (literals below) on tiny integer-valued buffers, with
# stand-in kernels written out in the test, so that a dropped auto-zero
# (P:141), an RW accumulate that loses the host value, an
# out-of-order execution or a mutated input fails one of them.
import numpy as np  # noqa: E402

from oracle.graph_model import serial_execute  # noqa: E402


def _k_vadd(t, arr):
    arr[2][...] = arr[0] + arr[1]


def _k_reduce(t, arr):          # @Atomic(ADD) result += sum
    arr[1][0] += arr[0].sum()


def _k_hist(t, arr):            # bins[k] += #{key = k}
    for k in arr[0]:
        if 0 <= k < arr[1].size:
            arr[1][k] += 1


KS = {"vadd": _k_vadd, "reduce": _k_reduce, "hist": _k_hist}


def test_serial_auto_zero_write_vs_readwrite():
    keys = np.array([0, 2, 2, 3, 7, -1], np.int32)   # 7 and -1 out of range
    host = {"k": keys, "bW": np.array([5, 5, 5, 5], np.int32),
            "bRW": np.array([5, 5, 5, 5], np.int32)}
    out = serial_execute([Task("hist", [Arg("k", READ), Arg("bW", WRITE)]),
                          Task("hist", [Arg("k", READ), Arg("bRW", READWRITE)])], host, KS)
    assert out["bW"].tolist() == [1, 0, 2, 1]        # W: auto-zeroed, then counted
    assert out["bRW"].tolist() == [6, 5, 7, 6]       # RW: host value + counts
    assert host["bW"].tolist() == [5, 5, 5, 5]       # the input state is not modified
    s = {"x": np.array([1.0, 2.0, 4.0]), "s": np.array([100.0]), "t": np.array([100.0])}
    out = serial_execute([Task("reduce", [Arg("x", READ), Arg("s", WRITE)]),
                          Task("reduce", [Arg("x", READ), Arg("t", READWRITE)])], s, KS)
    assert out["s"].tolist() == [7.0] and out["t"].tolist() == [107.0]


def test_serial_raw_chain_and_insertion_order():
    host = {"a": np.array([1.0, 2.0]), "b": np.array([10.0, 20.0]),
            "c": np.array([0.0, 0.0]), "d": np.array([0.0, 0.0]), "s": np.array([0.0])}
    # t0: c = a + b; t1: d = c + b (RAW on c); t2: s = sum(d) (RAW on d);
    # t3: c = a + a (WAR after t1 read c, WAW after t0) -- t1 must have seen
    # t0's c, not t3's.
    tasks = [Task("vadd", [Arg("a", READ), Arg("b", READ), Arg("c", WRITE)]),
             Task("vadd", [Arg("c", READ), Arg("b", READ), Arg("d", WRITE)]),
             Task("reduce", [Arg("d", READ), Arg("s", WRITE)]),
             Task("vadd", [Arg("a", READ), Arg("a", READ), Arg("c", WRITE)])]
    out = serial_execute(tasks, host, KS)
    assert out["d"].tolist() == [21.0, 42.0]
    assert out["s"].tolist() == [63.0]
    assert out["c"].tolist() == [2.0, 4.0]
    # reversed WAR pair: now t1 reads the LATER c
    out2 = serial_execute([tasks[0], tasks[3], tasks[1]], host, KS)
    assert out2["d"].tolist() == [12.0, 24.0]


def test_serial_read_read_independent_and_accumulate_order():
    host = {"x": np.array([3.0, 4.0]), "s": np.array([1.0]), "t": np.array([0.0])}
    # two readers of x in either order give the same result (no edge, R9)
    t_s = Task("reduce", [Arg("x", READ), Arg("s", READWRITE)])
    t_t = Task("reduce", [Arg("x", READ), Arg("t", WRITE)])
    for order in ([t_s, t_t], [t_t, t_s]):
        out = serial_execute(order, host, KS)
        assert out["s"].tolist() == [8.0] and out["t"].tolist() == [7.0]
        assert out["x"].tolist() == [3.0, 4.0]
    # RW accumulates across tasks (1 + 7 + 7); a W in between restarts at 0
    out = serial_execute([t_s, t_s], host, KS)
    assert out["s"].tolist() == [15.0]
    out = serial_execute([t_s, Task("reduce", [Arg("x", READ), Arg("s", WRITE)]), t_s], host, KS)
    assert out["s"].tolist() == [14.0]
