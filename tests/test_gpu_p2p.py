"""JACC_GRAPH_P2P: collectives over peer memory, fused into their producers.

World 1 exercises every kernel path against the local window; world 2 runs
two processes on the box's single GPU that map each other's windows through
CUDA IPC -- the same cudaIpcOpenMemHandle / peer-store / flag protocol the
N-GPU run uses over NVLink, with the two contexts time-sliced on one device.
Results are compared with the oracle (bitwise for histogram, all-gather,
broadcast and the N-body shards; 1e-4 sum|x| for the float sums) and with
the single-GPU graph.
"""
import os
import sys

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
J = pytest.importorskip("paper_1508_06791_b200")
from paper_1508_06791_b200 import jacc  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R, W, RW = 1, 2, 3


def pinned(a):
    """numpy view of a pinned host copy of `a` (capturable H2D/D2H for replay)."""
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    v = t.numpy()
    assert v.base is not None
    return v


def _collective_graph(g, rank, world, keys, x, big, pos_shard, bc):
    """hist -> allreduce (fused), reduce -> allreduce (fused), a large
    standalone f32 allreduce, a standalone allgather, a broadcast from the
    last rank.  Returns the output buffers (host buffers pinned)."""
    from paper_1508_06791_b200.torch_glue import peer_tensor
    bins = pinned(np.zeros(256, np.int32))
    s = pinned(np.zeros(1, np.float32))
    gathered = pinned(np.zeros((pos_shard.shape[0] * world, 4), np.float32))
    bct = peer_tensor(g, (bc.size,))
    bct.copy_(torch.from_numpy(bc if rank == world - 1 else np.zeros_like(bc)))
    g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, R), g.a(bins, W)], jacc.jacc_hist_params_t(256))
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(bins, RW)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(x, R), g.a(s, W)])
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(s, RW)])
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(big, RW)])
    g.add_task(J.JACC_OP_ALLGATHER, [g.a(pos_shard, R, f32x4=True), g.a(gathered, W, f32x4=True)])
    g.add_task(J.JACC_OP_BROADCAST, [g.a(bct, RW)], jacc.jacc_bcast_params_t(world - 1))
    return bins, s, gathered, bct


def _nbody_chain(g, pos, vel, lo, hi, steps, world):
    """The bench's N>1 N-body shape: allgather(L[k%2] -> ALL), nbody(ALL ->
    L[(k+1)%2]); ALL is a DEVICE buffer in the window."""
    from paper_1508_06791_b200.torch_glue import peer_tensor
    n = pos.shape[0]
    prm = jacc.jacc_nbody_params_t(lo, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G)
    L = [pinned(pos[lo:hi]), pinned(np.zeros((hi - lo, 4), np.float32))]
    V = pinned(vel[lo:hi])
    ALL = peer_tensor(g, (n, 4))
    for k in range(steps):
        g.add_task(J.JACC_OP_ALLGATHER, [g.a(L[k % 2], R, True, f32x4=True), g.a(ALL, W, f32x4=True)])
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(ALL, R, f32x4=True), g.a(V, RW, True, f32x4=True),
                                               g.a(L[(k + 1) % 2], W, True, f32x4=True)], prm)
    return L, V


def _single_gpu_nbody(pos, vel, steps):
    from paper_1508_06791_b200.torch_glue import make_graph
    g, _ = make_graph(0)
    P = [pos.copy(), np.zeros_like(pos)]
    V = vel.copy()
    prm = jacc.jacc_nbody_params_t(0, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G)
    for k in range(steps):
        g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(P[k % 2], R, f32x4=True), g.a(V, RW, f32x4=True),
                                              g.a(P[(k + 1) % 2], W, f32x4=True)], prm)
    g.run()
    g.destroy()
    return P[steps % 2], V


@pytest.mark.parametrize("flags", [0, J.JACC_GRAPH_REPLAY])
def test_p2p_world1(flags):
    from paper_1508_06791_b200.torch_glue import make_graph
    torch.cuda.set_device(0)
    g, _ = make_graph(0, flags=J.JACC_GRAPH_P2P | flags)
    keys = pinned(synth.hist_keys((1 << 20) + 5, seed=21))
    x = pinned(synth.uniform_f32(99999, 22))
    big0 = synth.uniform_f32(300000, 23)
    big = pinned(big0)
    pos, _ = synth.nbody_state(1024, seed=24)
    pos = pinned(pos)
    bc = np.arange(1000, dtype=np.float32)
    bins, s, gathered, bct = _collective_graph(g, 0, 1, keys, x, big, pos, bc)
    for it in range(3):   # three epochs of every slot (both staging parities)
        big[:] = big0
        g.run()
        assert np.array_equal(bins, oracle.histogram(keys, 256)), it
        ref, absum = oracle.reduce_sum(x)
        assert abs(s[0] - ref) <= 1e-4 * absum, it
        assert np.array_equal(big, big0), it            # world 1: the sum over one rank
        assert np.array_equal(gathered, pos), it
        assert np.array_equal(bct.cpu().numpy(), bc), it
    st = g.stats()
    # 7 tasks: hist+allreduce and reduce+allreduce fused -> 5 kernels (+2 for the big allreduce's 2 phases)
    assert st["collectives"] == 5 and st["kernels"] == 2, st
    assert st["launches"] == 6, st
    if flags & J.JACC_GRAPH_REPLAY:
        assert st["graph_captures"] == 1 and st["graph_replays"] == 2, st
    g.destroy()


def test_p2p_world1_nbody_bitwise():
    """P2P N-body chain (standalone allgather, then nbody+allgather fused)
    at world 1 == the plain single-graph chain, bitwise."""
    from paper_1508_06791_b200.torch_glue import make_graph
    torch.cuda.set_device(0)
    n, steps = 4096, 4
    pos, vel = synth.nbody_state(n, seed=12)
    g, _ = make_graph(0, flags=J.JACC_GRAPH_P2P)
    L, V = _nbody_chain(g, pos, vel, 0, n, steps, 1)
    g.run()
    st = g.stats()
    assert (st["h2d_count"], st["d2h_count"]) == (2, 3)
    # 1 standalone allgather + steps x (partial + finish with the fused allgather)
    assert st["launches"] == 1 + 2 * steps, st
    g.destroy()
    P1, V1 = _single_gpu_nbody(pos, vel, steps)
    assert np.array_equal(L[steps % 2], P1) and np.array_equal(V, V1)


def test_p2p_requires_window_buffer():
    from paper_1508_06791_b200.torch_glue import make_graph
    g, _ = make_graph(0, flags=J.JACC_GRAPH_P2P)
    send = np.zeros((16, 4), np.float32)
    recv = torch.zeros((16, 4), device="cuda")     # a DEVICE buffer outside the window
    g.add_task(J.JACC_OP_ALLGATHER, [g.a(send, R, f32x4=True), g.a(recv, W, f32x4=True)])
    with pytest.raises(J.JaccError, match="INVALID_ARG"):
        g.run()
    g.destroy()


# ---------------------------------------------------------------- world 2
def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)       # both ranks share the box's one GPU
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        import paper_1508_06791_b200 as J
        from paper_1508_06791_b200.torch_glue import make_graph, peer_setup
        res = {}
        for flags in (0, J.JACC_GRAPH_REPLAY):
            g, _ = make_graph(0, rank=rank, world=world, flags=J.JACC_GRAPH_P2P | flags)
            peer_setup(g, 32 << 20)
            keys = synth.hist_keys((1 << 20) + 6, seed=31)
            lo, hi = synth.shard_range(keys.size, rank, world)
            x = synth.uniform_f32(200001, 32)
            xl, xh = synth.shard_range(x.size, rank, world)
            bigs = [synth.uniform_f32(300000, 40 + r) for r in range(world)]
            big = pinned(bigs[rank])
            pos, vel = synth.nbody_state(2048, seed=33)
            pl, ph = synth.shard_range(pos.shape[0], rank, world)
            bc = np.arange(1000, dtype=np.float32) * 3
            kshard = pinned(keys[lo:hi])
            xshard = pinned(x[xl:xh])
            bins, s, gathered, bct = _collective_graph(g, rank, world, kshard, xshard, big, pinned(pos[pl:ph]), bc)
            L, V = _nbody_chain(g, pos, vel, pl, ph, 3, world)
            ok = {}
            for it in range(3):
                big[:] = bigs[rank]
                g.run()
                ref, absum = oracle.reduce_sum(x)
                big_ref = bigs[0].astype(np.float32)
                for r in range(1, world):                    # rank order, fp32 adds
                    big_ref = big_ref + bigs[r].astype(np.float32)
                ok[it] = dict(hist=bool(np.array_equal(bins, oracle.histogram(keys, 256))),
                              reduce=bool(abs(s[0] - ref) <= 1e-4 * absum),
                              big=bool(np.array_equal(big, big_ref)),
                              gather=bool(np.array_equal(gathered, pos)),
                              bcast=bool(np.array_equal(bct.cpu().numpy(), bc)))
                if it == 0:
                    ok["pos"] = L[3 % 2].copy()
                    ok["vel"] = V.copy()
            st = g.stats()
            ok["replays"] = int(st["graph_replays"])
            res[flags] = ok
            g.destroy()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_p2p_world2_one_gpu(world):
    """world ranks = world processes time-sliced on the box's one GPU."""
    import torch.multiprocessing as mp
    port = 29700 + (os.getpid() % 200) + 7 * world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    pos, vel = synth.nbody_state(2048, seed=33)
    P1, V1 = _single_gpu_nbody(pos, vel, 3)
    for r in range(world):
        assert "error" not in out[r], out[r].get("error")
        for flags, ok in out[r].items():
            # CACHABLE inputs change the plan after execute 1 (H2D elided): capture, re-capture, replay
            assert ok["replays"] == (1 if flags else 0), (r, flags, ok["replays"])
            for it in range(3):
                assert all(ok[it].values()), (r, flags, it, ok[it])
            lo, hi = synth.shard_range(2048, r, world)
            # shard invariance: the 2-rank chain equals the 1-GPU chain bitwise
            assert np.array_equal(ok["pos"], P1[lo:hi]), (r, flags)
            assert np.array_equal(ok["vel"], V1[lo:hi]), (r, flags)


def _swap_worker(rank, world, port, q):
    """N-body step whose targets are the OTHER rank's shard (tgt_offset !=
    rank * n_tgt) with the all-gather's receive buffer = the step's pos_src:
    the runtime must not fuse the all-gather into the finish kernel (peers
    would overwrite slots it still reads); it runs standalone."""
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        import paper_1508_06791_b200 as J
        from paper_1508_06791_b200.torch_glue import make_graph, peer_setup, peer_tensor
        n = 2048
        pos, vel = synth.nbody_state(n, seed=34)
        vel[:, :3] = synth.rng(35).standard_normal((n, 3)).astype(np.float32) * 0.1
        res = {}
        for swap in (True, False):
            g, _ = make_graph(0, rank=rank, world=world, flags=J.JACC_GRAPH_P2P)
            peer_setup(g, 8 << 20)
            other = (rank + 1) % world if swap else rank
            lo, hi = synth.shard_range(n, rank, world)
            tlo, thi = synth.shard_range(n, other, world)
            ALL = peer_tensor(g, (n, 4))
            L0 = pinned(pos[lo:hi]); L1 = pinned(np.zeros((thi - tlo, 4), np.float32))
            V = pinned(vel[tlo:thi])
            prm = jacc.jacc_nbody_params_t(tlo, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G)
            g.add_task(J.JACC_OP_ALLGATHER, [g.a(L0, R, f32x4=True), g.a(ALL, W, f32x4=True)])
            g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(ALL, R, f32x4=True), g.a(V, RW, f32x4=True),
                                                   g.a(L1, W, f32x4=True)], prm)
            g.add_task(J.JACC_OP_ALLGATHER, [g.a(L1, R, f32x4=True), g.a(ALL, W, f32x4=True)])
            g.run()
            res[swap] = dict(all=ALL.cpu().numpy().copy(), vel=V.copy(), launches=g.stats()["launches"])
            g.destroy()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


def test_p2p_nbody_gather_not_fused_when_unsafe():
    import torch.multiprocessing as mp
    world, n = 2, 2048
    port = 29600 + (os.getpid() % 90)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_swap_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    pos, vel = synth.nbody_state(n, seed=34)
    vel[:, :3] = synth.rng(35).standard_normal((n, 3)).astype(np.float32) * 0.1
    P1, V1 = _single_gpu_nbody(pos, vel, 1)
    sh = [synth.shard_range(n, r, world) for r in range(world)]
    for r in range(world):
        assert "error" not in out[r], out[r].get("error")
        sw, al = out[r][True], out[r][False]
        # swapped: slot q of ALL holds rank q's targets = shard (q + 1) % world
        want = np.concatenate([P1[slice(*sh[(q + 1) % world])] for q in range(world)])
        assert np.array_equal(sw["all"], want), r
        assert np.array_equal(sw["vel"], V1[slice(*sh[(r + 1) % world])]), r
        assert np.array_equal(al["all"], P1) and np.array_equal(al["vel"], V1[slice(*sh[r])]), r
        # aligned: gather, partial, finish+gather (3); swapped: + a standalone gather (4)
        assert (al["launches"], sw["launches"]) == (3, 4), (al["launches"], sw["launches"])


def _halo_worker(rank, world, port, q, cases):
    """2D convolution sharded by row bands: each rank holds
    its band, exchanges r halo rows with its neighbours over the peer windows
    (JACC_OP_HALO_EXCHANGE_F32) and convolves its extended band
    (JACC_CONV2D_HALO_ROWS); three epochs (both staging parities)."""
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        import paper_1508_06791_b200 as J
        from paper_1508_06791_b200 import jacc
        from paper_1508_06791_b200.torch_glue import make_graph, peer_setup
        res = {}
        for (H, Wd, r, flags) in cases:
            img = synth.uniform_f32(H * Wd, 710 + H, -1, 1).reshape(H, Wd)
            f = synth.uniform_f32((2 * r + 1) ** 2, 711, -1, 1).reshape(2 * r + 1, 2 * r + 1)
            lo, hi = synth.shard_range(H, rank, world)
            g, _ = make_graph(0, rank=rank, world=world, flags=J.JACC_GRAPH_P2P | flags)
            peer_setup(g, 4 << 20)
            band = pinned(img[lo:hi])
            ext = pinned(np.zeros((hi - lo + 2 * r, Wd), np.float32))
            out = pinned(np.zeros((hi - lo, Wd), np.float32))
            g.add_task(J.JACC_OP_HALO_EXCHANGE_F32, [g.a(band, R), g.a(ext, W)],
                       jacc.jacc_halo_params_t(hi - lo, Wd, r, 0))
            g.add_task(J.JACC_OP_CONV2D_F32, [g.a(ext, R), g.a(f, R), g.a(out, W)],
                       jacc.jacc_conv2d_params_t(hi - lo, Wd, r, J.JACC_CONV2D_HALO_ROWS))
            outs = []
            for it in range(3):
                g.run()
                outs.append((ext.copy(), out.copy()))
            res[(H, Wd, r, flags)] = (outs, g.stats()["launches"])
            g.destroy()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception:
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_p2p_conv2d_row_bands(world):
    """Every rank's halo rows equal oracle.halo_band and its output rows equal
    the single-GPU convolution of the whole image bit for bit (same kernel,
    same per-pixel sum order), three epochs, direct and replayed."""
    import torch.multiprocessing as mp
    from paper_1508_06791_b200.torch_glue import make_graph
    cases = [(1030, 256, 2, 0), (515, 250, 2, J.JACC_GRAPH_REPLAY), (2048, 2048, 2, 0), (90, 72, 4, 0)]
    port = 29500 + (os.getpid() % 90) + 3 * world
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, qu, cases)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(qu.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for (H, Wd, r, flags) in cases:
        img = synth.uniform_f32(H * Wd, 710 + H, -1, 1).reshape(H, Wd)
        f = synth.uniform_f32((2 * r + 1) ** 2, 711, -1, 1).reshape(2 * r + 1, 2 * r + 1)
        full = np.zeros_like(img)
        g, _ = make_graph(0)
        g.add_task(J.JACC_OP_CONV2D_F32, [g.a(img, R), g.a(f, R), g.a(full, W)],
                   jacc.jacc_conv2d_params_t(H, Wd, r, 0))
        g.run()
        g.destroy()
        ref, ab = oracle.conv2d(img, f)
        assert np.all(np.abs(full.astype(np.float64) - ref) <= 1e-5 * ab + 1e-30)
        for rk in range(world):
            assert "error" not in out[rk], out[rk].get("error")
            outs, launches = out[rk][(H, Wd, r, flags)]
            lo, hi = synth.shard_range(H, rk, world)
            for it, (ext, o) in enumerate(outs):
                assert np.array_equal(ext, oracle.halo_band(img, lo, hi, r)), (H, rk, it)
                assert np.array_equal(o, full[lo:hi]), (H, rk, it)


def test_p2p_window_errors():
    """Error paths of the peer windows (include/jacc.h): a full window is
    JACC_ERR_OOM, handles whose window sizes differ are JACC_ERR_INVALID_ARG
    (checked before any IPC mapping), a second init is JACC_ERR_STATE."""
    from paper_1508_06791_b200.torch_glue import make_graph
    g, _ = make_graph(0, flags=J.JACC_GRAPH_P2P)
    h = g.peer_init(512 << 10)                 # 256 KiB flag header + 256 KiB heap
    with pytest.raises(J.JaccError, match="STATE"):
        g.peer_init(0)
    assert g.peer_alloc(200 << 10)
    with pytest.raises(J.JaccError, match="OOM"):
        g.peer_alloc(200 << 10)
    g.destroy()
    g, _ = make_graph(0, rank=0, world=2, flags=J.JACC_GRAPH_P2P)
    h0 = g.peer_init(1 << 20)
    h1 = jacc.jacc_peer_handle_t.from_buffer_copy(bytes(h0))
    h1.rank, h1.window_bytes = 1, 2 << 20
    with pytest.raises(J.JaccError, match="INVALID_ARG"):
        g.peer_connect([h0, h1])
    with pytest.raises(J.JaccError, match="INVALID_ARG"):
        g.peer_connect([h1, h0])               # handles out of rank order
    g.destroy()


def test_p2p_collective_slot_limit():
    """Every collective task owns a flag slot; one slot is reserved for the
    teardown barrier, so a P2P graph takes at most 1023 collective tasks."""
    from paper_1508_06791_b200.torch_glue import make_graph
    g, _ = make_graph(0, flags=J.JACC_GRAPH_P2P)
    x = np.ones(4, np.float32)
    for _ in range(1023):
        g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(x, RW)])
    g.run()
    assert np.array_equal(x, np.ones(4, np.float32))       # world 1: identity, 1023 times
    g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(x, RW)])
    with pytest.raises(J.JaccError, match="UNSUPPORTED"):
        g.run()
    g.destroy()
