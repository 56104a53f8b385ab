"""Parity of the graph bench.py times, in the launch configuration it times
(task ③ "at BASELINE.json's full sizes, in the launch
configuration bench.py times"): the jacc-suite graph at full size, both the
device-resident form (JACC_GRAPH_SERIAL, the timed region) and the pinned
host-buffer form (4 compute streams, the e2e region), checked against the
oracle on EVERY output (cfg1-3 vs the oracle, the 8192^3 C element by
element, all 2^17 bodies after the 10 steps); and the two forms must agree
bit for bit (schedule invariance of every kernel).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
J = pytest.importorskip("paper_1508_06791_b200")
from paper_1508_06791_b200 import jacc  # noqa: E402

import bench  # noqa: E402


def _np(t):
    return t.cpu().numpy() if t.is_cuda else t.numpy()


@pytest.fixture(scope="module")
def suite_outputs():
    outs = {}
    # "device" = the timed region's configuration (one stream, plan replay:
    # the first execute captures the action list and launches the graph)
    for form, host, flags in (("device", False, J.JACC_GRAPH_SERIAL | J.JACC_GRAPH_REPLAY), ("host", True, 0)):
        s = bench.Suite(torch, J, jacc, 0, 1, 0, host_mode=host, sgemm_mode=J.JACC_SGEMM_3XTF32, flags=flags)
        s.g.run()
        st = s.g.stats()
        if form == "device":
            assert st["graph_captures"] == 1, st
        outs[form] = ({k: _np(v).copy() for k, v in s.out.items()}, st)
        s.g.destroy()
        del s
        torch.cuda.empty_cache()
    return outs


def test_suite_forms_bitwise_equal(suite_outputs):
    dev, _ = suite_outputs["device"]
    host, st = suite_outputs["host"]
    for k in dev:
        assert np.array_equal(dev[k], host[k]), k
    # host form: every input copied in once, every output out once (SURVEY count table)
    assert st["h2d_count"] == 8 and st["d2h_count"] == 9


def test_suite_cfg1_cfg2(suite_outputs):
    o, _ = suite_outputs["device"]
    a, b = synth.vadd_inputs()
    c = oracle.vadd(a, b)
    assert np.array_equal(o["c"], c)
    ref, absum = oracle.reduce_sum(c)
    assert abs(float(o["s"][0]) - ref) <= 1e-4 * absum
    keys = synth.hist_keys()
    assert np.array_equal(o["bins"], oracle.histogram(keys, 256))


def test_suite_cfg3_full(suite_outputs):
    """Black-Scholes, every one of the 2^26 options against the fp64 oracle
    (R12 gate)."""
    o, _ = suite_outputs["device"]
    u = synth.bs_rand()
    oc, op = oracle.blackscholes(u)
    uu = u.astype(np.float64)
    S = 10 * uu + 100 * (1 - uu); T = uu + 10 * (1 - uu); Rr = 0.01 * uu + 0.05 * (1 - uu)
    scale = S + S * np.exp(-Rr * T)          # S + K e^{-RT}, K = S (R12)
    assert np.max(np.abs(o["call"] - oc) / scale) <= 1e-5
    assert np.max(np.abs(o["put"] - op) / scale) <= 1e-5


@pytest.mark.slow
def test_suite_cfg4_full_elementwise(suite_outputs):
    """SGEMM 8192^3 on U[0,1) inputs: EVERY element of C against the full
    fp64 oracle (gate M1: max elementwise relative error <= 1e-4)."""
    o, _ = suite_outputs["device"]
    n = synth.CFG4_MNK
    A, B = synth.sgemm_inputs(n, n, n)
    R = oracle.sgemm_rows(A, B)
    rel = np.abs(o["C"] - R) / np.abs(R)
    assert rel.max() <= 1e-4, rel.max()


@pytest.mark.slow
def test_suite_cfg5_full_oracle(suite_outputs):
    """10 steps of 2^17 bodies, EVERY body against the fp64 oracle's 10
    steps (north_star gates: |dx_i| <= 1e-4 R with R = 1 the ball radius,
    |dv_i| <= 1e-4 mean|v|), plus the invariants: momentum conserved
    (sum m v = 0 from rest), masses carried unchanged, every body moved by at
    most |v|max * 10 * dt."""
    o, _ = suite_outputs["device"]
    pos0, vel0 = synth.nbody_state()
    op, ov = oracle.nbody_steps(pos0, vel0, synth.CFG5_STEPS, synth.NBODY_DT, synth.NBODY_EPS2,
                                synth.NBODY_G)
    pos, vel = o["pos"].astype(np.float64), o["vel"].astype(np.float64)
    dx = np.max(np.abs(pos[:, :3] - op[:, :3]))
    vs = np.mean(np.linalg.norm(ov[:, :3], axis=1))
    dv = np.max(np.abs(vel[:, :3] - ov[:, :3]))
    assert dx <= 1e-4 and dv <= 1e-4 * vs, (dx, dv / vs)
    m = pos0[:, 3:4].astype(np.float64)
    p_tot = np.sum(m * vel[:, :3], axis=0)
    assert np.max(np.abs(p_tot)) <= 1e-5 * np.sum(m * np.abs(vel[:, :3]))
    assert np.array_equal(o["pos"][:, 3], pos0[:, 3])
    vmax = np.max(np.linalg.norm(vel[:, :3], axis=1))
    disp = np.linalg.norm(pos[:, :3] - pos0[:, :3].astype(np.float64), axis=1)
    assert np.all(np.isfinite(pos)) and np.max(disp) <= vmax * synth.CFG5_STEPS * synth.NBODY_DT * 1.0001


# ------------------------------------------------------------------ world 2
def _suite_worker(rank, world, port, q):
    """One rank of the bench's N>1 graph (P2P collectives, the timed launch
    configuration), both ranks on the box's one GPU."""
    try:
        import os
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, root)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        import paper_1508_06791_b200 as J
        from paper_1508_06791_b200 import jacc
        s = bench.Suite(torch, J, jacc, rank, world, 0, host_mode=False, sgemm_mode=J.JACC_SGEMM_3XTF32,
                        flags=J.JACC_GRAPH_SERIAL | J.JACC_GRAPH_REPLAY, p2p=True)
        for _ in range(2):      # capture, then replay (the N-body state advances: keep the first)
            s.g.run()
            if _ == 0:
                out = {k: (v.cpu().numpy() if v.is_cuda else v.numpy()).copy() for k, v in s.out.items()}
        st = s.g.stats()
        s.g.destroy()
        del s
        torch.cuda.empty_cache()
        # the e2e (host-buffer) form: B copied in as 1/world row blocks and
        # all-gathered over the peer windows before the SGEMM
        h = bench.Suite(torch, J, jacc, rank, world, 0, host_mode=True, sgemm_mode=J.JACC_SGEMM_3XTF32, p2p=True)
        h.g.run()
        hst = h.g.stats()
        hout = {k: (v.cpu().numpy() if v.is_cuda else v.numpy()).copy() for k, v in h.out.items()}
        h.g.destroy()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, {"out": out, "replays": int(st["graph_replays"]), "host_out": hout,
                      "host_h2d_bytes": int(hst["h2d_bytes"]), "host_tasks": sorted(h.tasks)}))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


@pytest.mark.slow
def test_suite_world2_p2p(suite_outputs):
    """The bench's N = 2 graph at full size: every rank's shard against the
    oracle (histogram and all-reduced bins bitwise, sums within tolerance)
    and bitwise against the 1-GPU suite where the decomposition promises it
    (vadd, Black-Scholes, SGEMM rows, N-body after 10 all-gathered steps)."""
    import os
    import torch.multiprocessing as mp
    world = 2
    port = 29900 + (os.getpid() % 90)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_suite_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    one, _ = suite_outputs["device"]
    keys = synth.hist_keys()
    bins_ref = oracle.histogram(keys, 256)
    a, b = synth.vadd_inputs()
    ref_s, absum = oracle.reduce_sum(oracle.vadd(a, b))
    for r in range(world):
        assert "error" not in res[r], res[r].get("error")
        o = res[r]["out"]
        assert res[r]["replays"] == 1
        assert np.array_equal(o["bins"], bins_ref)                       # allreduce of the shards' bins
        assert abs(float(o["s"][0]) - ref_s) <= 1e-4 * absum             # allreduce of partial sums
        lo, hi = synth.shard_range(synth.CFG1_N, r, world)
        assert np.array_equal(o["c"], one["c"][lo:hi])
        lo, hi = synth.shard_range(synth.CFG3_N, r, world)
        assert np.array_equal(o["call"], one["call"][lo:hi]) and np.array_equal(o["put"], one["put"][lo:hi])
        lo, hi = synth.shard_range(synth.CFG4_MNK, r, world)
        assert np.array_equal(o["C"], one["C"][lo:hi])
        lo, hi = synth.shard_range(synth.CFG5_N, r, world)
        assert np.array_equal(o["pos"], one["pos"][lo:hi]) and np.array_equal(o["vel"], one["vel"][lo:hi])
        # host-buffer form: the same results, B arriving by all-gather
        assert "allgather_B" in res[r]["host_tasks"]
        for k in o:
            assert np.array_equal(res[r]["host_out"][k], o[k]), k
        # H2D per rank = its shards only: a, b, keys, u, A rows, B ROWS (not all of B), positions, velocities
        def span(n):
            l, h = synth.shard_range(n, r, world)
            return h - l
        n4 = synth.CFG4_MNK
        want = (2 * 4 * span(synth.CFG1_N) + 4 * span(synth.CFG2_N) + 4 * span(synth.CFG3_N) +
                4 * span(n4) * n4 * 2 + 16 * span(synth.CFG5_N) * 2)
        assert res[r]["host_h2d_bytes"] == want, (res[r]["host_h2d_bytes"], want)
