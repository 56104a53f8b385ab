"""GPU task-graph semantics through the C-ABI (§2.3, P:286-290;
SURVEY §8(c)-G): counted copies, elimination soundness (naive == elided
outputs), serializability against the oracle's serial executor on random
DAGs, cross-execute residency (CACHABLE, invalidate), failure atomicity and
out-of-order issue of independent tasks.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import graph_model as gm

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
J = pytest.importorskip("paper_1508_06791_b200")
from paper_1508_06791_b200 import jacc  # noqa: E402
from paper_1508_06791_b200.torch_glue import make_graph  # noqa: E402

R, W, RW = J.JACC_READ, J.JACC_WRITE, J.JACC_READWRITE


def _graph(**kw):
    return make_graph(0, **kw)[0]


def test_cfg1_counted_copies_and_values():
    n = synth.CFG1_N
    a, b = synth.vadd_inputs()
    c = np.zeros(n, np.float32); s = np.zeros(1, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R, True), g.a(b, R, True), g.a(c, W)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
    g.run()
    st = g.stats()
    assert (st["h2d_count"], st["d2h_count"], st["memsets"], st["kernels"]) == (2, 2, 1, 2)
    assert st["h2d_bytes"] == 8 * n and st["d2h_bytes"] == 4 * n + 4
    ref_c = oracle.vadd(a, b)
    assert np.array_equal(c, ref_c)
    ref, absum = oracle.reduce_sum(ref_c)
    assert abs(s[0] - ref) <= 1e-4 * absum
    # 2nd execute: a, b resident (CACHABLE) -> no H2D; same results
    c[:] = 0; s[:] = 0
    g.run()
    st = g.stats()
    assert (st["h2d_count"], st["d2h_count"]) == (0, 2)
    assert np.array_equal(c, ref_c)
    # host writes a -> invalidate -> exactly one H2D again
    a[:] = 1.0
    g.invalidate(a)
    g.run()
    st = g.stats()
    assert (st["h2d_count"], st["h2d_bytes"]) == (1, 4 * n)
    assert np.array_equal(c, oracle.vadd(a, b))
    g.destroy()


@pytest.mark.parametrize("flags", [0, "merge_replay", "merge_replay_notiming"])
def test_cfg1_k_iterations_one_graph(flags):
    """Paper protocol (SURVEY §8(c)-G row 'cfg1 xK'): K iterations of
    vadd -> reduce in ONE graph cost a single H2D per input and a single D2H
    per output (naive: 3K / 2K), and the final values equal one iteration's."""
    if flags == "merge_replay":
        flags = J.JACC_GRAPH_MERGE | J.JACC_GRAPH_REPLAY
    elif flags == "merge_replay_notiming":
        flags = J.JACC_GRAPH_MERGE | J.JACC_GRAPH_REPLAY | J.JACC_GRAPH_NO_TIMING
    n, K = 1 << 16, 40
    a, b = synth.vadd_inputs(n, seed=5)
    c = np.zeros(n, np.float32); s = np.zeros(1, np.float32)
    g = _graph(flags=flags)
    for _ in range(K):
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
    for _ in range(2):   # second run exercises the replayed plan
        c[:] = 0; s[:] = 0
        g.run()
        st = g.stats()
        assert (st["h2d_count"], st["d2h_count"]) == (2, 2)
        if not flags:
            assert st["kernels"] == 2 * K
        ref_c = oracle.vadd(a, b)
        assert np.array_equal(c, ref_c)
        ref, absum = oracle.reduce_sum(ref_c)
        assert abs(s[0] - ref) <= 1e-4 * absum
    if flags & J.JACC_GRAPH_NO_TIMING:
        with pytest.raises(J.JaccError, match="STATE"):
            g.task_ms(0)
    else:
        assert g.task_ms(2 * K - 1) > 0
    g.destroy()
    gn = _graph(flags=J.JACC_GRAPH_NAIVE)
    for _ in range(K):
        gn.add_task(J.JACC_OP_VADD_F32, [gn.a(a, R), gn.a(b, R), gn.a(c, W)])
        gn.add_task(J.JACC_OP_REDUCE_SUM_F32, [gn.a(c, R), gn.a(s, W)])
    gn.run()
    st = gn.stats()
    assert (st["h2d_count"], st["d2h_count"]) == (3 * K, 2 * K)
    gn.destroy()


def test_naive_equals_elided_and_counts():
    n = 100003
    a, b = synth.vadd_inputs(n, seed=3)
    outs = {}
    for naive in (True, False):
        c = np.zeros(n, np.float32); d = np.zeros(n, np.float32); s = np.zeros(1, np.float32)
        g = _graph(flags=J.JACC_GRAPH_NAIVE if naive else 0)
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
        g.add_task(J.JACC_OP_VADD_F32, [g.a(c, R), g.a(b, R), g.a(d, W)])
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(d, R), g.a(s, W)])
        g.run()
        st = g.stats()
        outs[naive] = (c.copy(), d.copy(), s.copy(), st["h2d_bytes"] + st["d2h_bytes"])
        g.destroy()
    for x, y in zip(outs[True][:3], outs[False][:3]):
        assert np.array_equal(x, y)
    assert outs[False][3] < outs[True][3]   # optimized bytes strictly smaller


def _kernels_for_serial():
    def vadd(t, arr):
        arr[2][...] = oracle.vadd(arr[0], arr[1])

    def reduce(t, arr):
        s, _ = oracle.reduce_sum(arr[0], init=float(arr[1][0]))
        arr[1][0] = np.float32(s)

    def hist(t, arr):
        arr[1][...] = oracle.histogram(arr[0], arr[1].size, init=arr[1])

    def allreduce(t, arr):   # world == 1: identity
        pass

    def allgather(t, arr):
        arr[1][...] = arr[0]
    return {"vadd": vadd, "reduce": reduce, "hist": hist, "allreduce": allreduce, "allgather": allgather}


def test_serializability_random_dags():
    """50 random DAGs (3-8 tasks, random R/W modes) executed optimized and
    out of order == one-by-one insertion-order execution."""
    from test_abi_cpu import _Pool, _add, _random_tasks
    rng = np.random.default_rng(2024)
    kernels = _kernels_for_serial()
    done = 0
    while done < 50:
        tasks = _random_tasks(rng, int(rng.integers(3, 9)))
        if len(tasks) < 3:
            continue
        pool = _Pool(n=4099)
        allbufs = {**pool.f, **pool.s, **pool.k, **pool.h}
        for k, v in pool.f.items():
            v[:] = synth.uniform_f32(v.size, rng.integers(1 << 30))
        pool.k["K"][:] = rng.integers(-2, 18, pool.k["K"].size)
        for v in (pool.s["s"], pool.s["t"]):
            v[:] = rng.random()
        pool.h["H"][:] = rng.integers(0, 5, 16)
        host0 = {k: v.copy() for k, v in allbufs.items()}
        ref = gm.serial_execute(tasks, host0, kernels)
        g = _graph()
        for t in tasks:
            _add(g, pool, t)
        g.run()
        for k, v in allbufs.items():
            if k in ("s", "t"):
                # reduction outputs: fp32 tree vs fp64 oracle (R14); a RW
                # output also carries the accumulated host value
                scale = np.maximum(np.abs(ref[k]), 1.0) * 5e-5
                assert np.all(np.abs(v - ref[k]) <= scale), (k, tasks)
            else:
                # vadd / all-gather outputs (one RN fp32 add or a copy) and
                # integer bins are exact by construction: "exactly"
                assert np.array_equal(v, ref[k]), (k, tasks)
        g.destroy()
        done += 1


def test_state_machine_errors():
    """the graph executes atomically -- no structural change or second
    execute while EXECUTING; errors are status codes, never aborts."""
    n = 4096
    a, b = synth.vadd_inputs(n, seed=2)
    c = np.zeros(n, np.float32)
    g = _graph()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R, True), g.a(b, R), g.a(c, W)])
    g.execute()
    assert g.stats()["state"] == 1                       # EXECUTING
    with pytest.raises(J.JaccError) as e:
        g.execute()
    assert e.value.status == J.JACC_ERR_STATE
    with pytest.raises(J.JaccError) as e:
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
    assert e.value.status == J.JACC_ERR_STATE
    with pytest.raises(J.JaccError) as e:
        g.invalidate(a)
    assert e.value.status == J.JACC_ERR_STATE
    g.sync()
    assert g.stats()["state"] == 2                       # DONE
    assert np.array_equal(c, oracle.vadd(a, b))
    with pytest.raises(J.JaccError) as e:
        g.invalidate(np.zeros(3, np.float32))
    assert e.value.status == J.JACC_ERR_NOT_FOUND
    # DONE graphs are re-executable and can grow (state back to BUILDING)
    s = np.zeros(1, np.float32)
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
    assert g.stats()["state"] == 0
    g.run()
    ref, absum = oracle.reduce_sum(c)
    assert abs(s[0] - ref) <= 1e-4 * absum
    g.destroy()


def test_failure_leaves_host_untouched():
    n = 65536
    a, b = synth.vadd_inputs(n, seed=1)
    c = np.full(n, 3.0, np.float32); s = np.full(1, 5.0, np.float32)
    c0, s0 = c.copy(), s.copy()
    g = _graph(fail_task=2)   # issuing task 1 fails
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
    with pytest.raises(J.JaccError) as e:
        g.run()
    assert e.value.status == J.JACC_ERR_INJECTED
    assert g.stats()["state"] == 3   # FAILED
    assert np.array_equal(c, c0) and np.array_equal(s, s0)
    g.destroy()


@pytest.mark.parametrize("flags", [0, J.JACC_GRAPH_REPLAY])
def test_failed_execute_drops_residency(flags):
    """R8 + R5: a failed execute may already have run kernels that updated
    the device copies of CACHABLE RW/W buffers (here the velocity and the
    position ping-pong of an N-body chain); the host keeps the values of the
    last successful execute, so the next execute must upload them again
    instead of trusting the stale device copies."""
    n, steps = 3000, 3
    pos, vel = synth.nbody_state(n, seed=41)
    vel[:, :3] = synth.rng(42).standard_normal((n, 3)).astype(np.float32) * 0.1
    P = [pos.copy(), np.zeros_like(pos)]
    V = vel.copy()
    g = _graph(flags=flags)
    prm = jacc.jacc_nbody_params_t(0, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G)
    for k in range(steps):
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(P[k % 2], R, True, f32x4=True), g.a(V, RW, True, f32x4=True),
                                              g.a(P[(k + 1) % 2], W, True, f32x4=True)], prm)
    g.run()                                   # execute 1: everything resident afterwards
    host1 = [P[0].copy(), P[1].copy(), V.copy()]
    g.set_fail_task(3)                        # execute 2: steps 0 and 1 run, step 2 fails
    with pytest.raises(J.JaccError) as e:
        g.run()
    assert e.value.status == J.JACC_ERR_INJECTED
    assert all(np.array_equal(x, y) for x, y in zip((P[0], P[1], V), host1))
    g.set_fail_task(0)                        # execute 3 from the host state of execute 1
    g.run()
    st = g.stats()
    assert st["h2d_count"] == 2, st           # P[0] and V re-uploaded, not taken as resident
    g.destroy()
    # reference: a fresh graph from execute 1's host state
    P2 = [host1[0].copy(), host1[1].copy()]
    V2 = host1[2].copy()
    g = _graph()
    for k in range(steps):
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(P2[k % 2], R, f32x4=True), g.a(V2, RW, f32x4=True),
                                              g.a(P2[(k + 1) % 2], W, f32x4=True)], prm)
    g.run()
    g.destroy()
    assert np.array_equal(V, V2) and np.array_equal(P[steps % 2], P2[steps % 2])


def test_out_of_order_issue():
    """a task on DEVICE inputs does not wait for an unrelated
    task's large H2D: t1 (device inputs) completes before t0's inputs land."""
    big = 1 << 26   # 256 MiB per input
    a = torch.empty(big, dtype=torch.float32).pin_memory().uniform_()
    b = torch.empty(big, dtype=torch.float32).pin_memory().uniform_()
    c = torch.empty(big, dtype=torch.float32).pin_memory()
    x = torch.rand(1 << 20, device="cuda"); y = torch.rand(1 << 20, device="cuda")
    z = torch.empty(1 << 20, device="cuda")
    g, st = make_graph(0)
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
    g.add_task(J.JACC_OP_VADD_F32, [g.a(x, R), g.a(y, R), g.a(z, W)])
    streams = [int(l.split("stream=")[1].split()[0]) for l in g.dump().splitlines() if l.startswith("task")]
    assert streams[0] != streams[1]
    # warm-up execute: the first one allocates the device copies (torch's
    # caching allocator may cudaMalloc) and loads the kernels' module (lazy
    # loading), both of which can block the host thread for the length of
    # the copies; the second execute re-copies a and b (not CACHABLE)
    g.run()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_start.record(st["h2d"])
    g.execute()
    e_t1 = torch.cuda.Event(enable_timing=True)
    e_t1.record(st["compute"][streams[1]])      # after t1's kernel
    e_h2d = torch.cuda.Event(enable_timing=True)
    e_h2d.record(st["h2d"])                     # after both 256 MiB H2D copies
    g.sync()
    torch.cuda.synchronize()
    assert t_start.elapsed_time(e_t1) < t_start.elapsed_time(e_h2d)
    assert torch.equal(z, x + y)
    assert torch.equal(c[:4096], (a[:4096] + b[:4096]))
    g.destroy()


def test_plan_replay_cuda_graph():
    """JACC_GRAPH_REPLAY captures each distinct plan once into
    a CUDA graph and re-launches it; results equal the direct issue."""
    n = 1 << 20
    a = torch.from_numpy(synth.vadd_inputs(n)[0]).pin_memory()
    b = torch.from_numpy(synth.vadd_inputs(n)[1]).pin_memory()
    c = torch.zeros(n, dtype=torch.float32).pin_memory()
    s = torch.zeros(1, dtype=torch.float32).pin_memory()
    g = _graph(flags=J.JACC_GRAPH_REPLAY)
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R, True), g.a(b, R, True), g.a(c, W)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
    ref_c = oracle.vadd(a.numpy(), b.numpy())
    ref_s, absum = oracle.reduce_sum(ref_c)
    for i in range(4):
        c.zero_(); s.zero_()
        g.run()
        assert np.array_equal(c.numpy(), ref_c)
        assert abs(s.item() - ref_s) <= 1e-4 * absum
    st = g.stats()
    # plan 1 (with H2D of a, b) captured once; plan 2 (a, b resident) captured
    # once and replayed twice
    assert (st["graph_captures"], st["graph_replays"]) == (2, 2), st
    assert g.task_ms(0) > 0.0
    g.destroy()


def test_plan_replay_pageable_falls_back_to_direct_issue():
    n = 4099
    a, b = synth.vadd_inputs(n, seed=8)
    c = np.zeros(n, np.float32)
    g = _graph(flags=J.JACC_GRAPH_REPLAY)
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
    for _ in range(2):
        c[:] = 0
        g.run()
        assert np.array_equal(c, oracle.vadd(a, b))
    g.destroy()


@pytest.mark.parametrize("extra", [0, J.JACC_GRAPH_REPLAY])
def test_merge_vadd_reduce_bit_identical(extra):
    """P:289 "merge" (JACC_GRAPH_MERGE): vadd -> reduce issued as one fused
    kernel gives bit-identical c and s, the same counted copies, one launch."""
    n = (1 << 20) + 12
    a, b = synth.vadd_inputs(n, seed=21)
    outs = {}
    for flags in (0, J.JACC_GRAPH_MERGE | extra):
        ta = torch.from_numpy(a).pin_memory(); tb = torch.from_numpy(b).pin_memory()
        c = torch.zeros(n).pin_memory(); s = torch.zeros(1).pin_memory()
        g = _graph(flags=flags)
        g.add_task(J.JACC_OP_VADD_F32, [g.a(ta, R), g.a(tb, R), g.a(c, W)])
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
        for _ in range(2):
            g.run()
        st = g.stats()
        outs[flags] = (c.numpy().copy(), s.numpy().copy(), st)
        g.destroy()
    (c0, s0, st0), (c1, s1, st1) = outs[0], outs[J.JACC_GRAPH_MERGE | extra]
    assert np.array_equal(c0, c1) and np.array_equal(s0, s1)
    assert np.array_equal(c0, oracle.vadd(a, b))
    assert (st1["h2d_count"], st1["d2h_count"]) == (st0["h2d_count"], st0["d2h_count"])
    assert st0["launches"] == 2 and st1["launches"] == 1


def test_reduce_rw_accumulates_w_assigns():
    """@Atomic semantics: W auto-zeroes (the kernel stores the
    sum, no memset node), RW adds to the host value -- bitwise the sum + the
    prior value, whichever path."""
    x = synth.uniform_f32(70001, 9)
    ref = None
    for access, init in ((W, 123.0), (RW, 0.0), (RW, 5.5)):
        s = np.full(1, init, np.float32)
        g = _graph()
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s, access)])
        g.run()
        st = g.stats()
        assert st["memsets"] == (1 if access == W else 0)
        g.destroy()
        if ref is None:
            ref = s[0]
            r, absum = oracle.reduce_sum(x)
            assert abs(ref - r) <= 1e-4 * absum
        else:
            assert s[0] == np.float32(init) + ref     # one fp32 add of the same tree sum


def test_merge_p2p_triple_one_launch():
    """MERGE + P2P at world 1: vadd -> reduce -> allreduce(s) is ONE kernel
    (the fused vadd+reduce finishes the allreduce over the peer window), with
    results bitwise equal to the unmerged graph."""
    n = (1 << 20) + 40
    a, b = synth.vadd_inputs(n, seed=23)
    outs = {}
    for flags in (0, J.JACC_GRAPH_MERGE | J.JACC_GRAPH_P2P):
        c = np.zeros(n, np.float32); s = np.zeros(1, np.float32)
        g = _graph(flags=flags)
        g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(c, R), g.a(s, W)])
        g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(s, RW)])
        for _ in range(3):
            g.run()
        outs[flags] = (c.copy(), s.copy(), g.stats())
        g.destroy()
    (c0, s0, st0), (c1, s1, st1) = outs.values()
    assert np.array_equal(c0, c1) and np.array_equal(s0, s1)
    assert st1["launches"] == 1 and st1["collectives"] == 1, st1
