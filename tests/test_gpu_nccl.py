"""NCCL collective tasks through libjacc.so with torch's communicator.

The GPU box gives one GPU, so the collectives run with a world-size-1 NCCL
process group: this still exercises the whole plumbing the N>1 path uses --
ProcessGroupNCCL._comm_ptr() -> jacc_config_t.nccl_comm -> NCCL resolved with
dlsym from the libnccl.so torch loaded -> ncclAllReduce / ncclAllGather /
ncclBroadcast issued on the graph's comm stream, ordered by events against the
kernels that produce and consume the buffers.
"""
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
J = pytest.importorskip("paper_1508_06791_b200")
from paper_1508_06791_b200 import jacc  # noqa: E402


@pytest.fixture(scope="module")
def nccl_pg():
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(29400 + os.getpid() % 500))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    from paper_1508_06791_b200.torch_glue import nccl_comm_ptr
    ptr = nccl_comm_ptr()
    assert ptr != 0
    yield ptr
    dist.destroy_process_group()


def test_collectives_world1(nccl_pg):
    from paper_1508_06791_b200.torch_glue import make_graph
    R, W, RW = J.JACC_READ, J.JACC_WRITE, J.JACC_READWRITE
    g, _ = make_graph(0, world=1, nccl_comm=nccl_pg)
    keys = synth.hist_keys(1 << 20)
    bins = np.zeros(256, np.int32)
    x = synth.uniform_f32(1 << 16, 3)
    s = np.zeros(1, np.float32)
    pos, _ = synth.nbody_state(1024)
    gathered = np.zeros_like(pos)
    bc = np.arange(100, dtype=np.float32)
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(bins, W)], jacc.jacc_hist_params_t(256))
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(bins, RW)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s, W)])
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(s, RW)])
    g.add_task(J.JACC_OP_ALLGATHER, [g.a(pos, R, f32x4=True), g.a(gathered, W, f32x4=True)])
    g.add_task(J.JACC_OP_BROADCAST, [g.a(bc, RW)], jacc.jacc_bcast_params_t(0))
    g.run()
    st = g.stats()
    assert st["collectives"] == 4 and st["kernels"] == 2
    assert np.array_equal(bins, oracle.histogram(keys, 256))          # world 1: sum over one rank
    ref, absum = oracle.reduce_sum(x)
    assert abs(s[0] - ref) <= 1e-4 * absum
    assert np.array_equal(gathered, pos)
    assert np.array_equal(bc, np.arange(100, dtype=np.float32))
    g.destroy()


def test_nbody_spmd_shape_world1(nccl_pg):
    """The bench's N>1 N-body graph shape (allgather -> nbody on DEVICE temp)
    at world 1 equals the single-graph chain, bitwise."""
    from paper_1508_06791_b200.torch_glue import make_graph
    R, W, RW = J.JACC_READ, J.JACC_WRITE, J.JACC_READWRITE
    n, steps = 4096, 3
    pos, vel = synth.nbody_state(n, seed=12)
    prm = jacc.jacc_nbody_params_t(0, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G)
    g, _ = make_graph(0, world=1, nccl_comm=nccl_pg)
    L = [pos.copy(), np.zeros_like(pos)]
    V = vel.copy()
    ALL = torch.zeros((n, 4), dtype=torch.float32, device="cuda")
    for k in range(steps):
        g.add_task(J.JACC_OP_ALLGATHER, [g.a(L[k % 2], R, True, f32x4=True), g.a(ALL, W, f32x4=True)])
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(ALL, R, f32x4=True), g.a(V, RW, True, f32x4=True),
                                               g.a(L[(k + 1) % 2], W, True, f32x4=True)], prm)
    g.run()
    st = g.stats()
    assert (st["h2d_count"], st["d2h_count"]) == (2, 3)
    g.destroy()
    g2, _ = make_graph(0)
    P = [pos.copy(), np.zeros_like(pos)]
    V2 = vel.copy()
    for k in range(steps):
        g2.add_task(J.JACC_OP_NBODY_STEP_F32, [g2.a(P[k % 2], R, f32x4=True), g2.a(V2, RW, f32x4=True),
                                                g2.a(P[(k + 1) % 2], W, f32x4=True)], prm)
    g2.run()
    g2.destroy()
    assert np.array_equal(L[steps % 2], P[steps % 2]) and np.array_equal(V, V2)
