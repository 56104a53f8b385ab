"""Multi-process (world_size 2 and 4, gloo, CPU) checks of the N>1 path's host logic.

The GPU box used here has one GPU, so the SPMD decomposition bench.py uses at
N>1 is verified on CPU: every rank takes its shard
(synth.shard_range), computes it with the oracle, and the ranks combine with
the same collective the GPU path issues through NCCL (allreduce of partial
sums / bins, allgather of N-body positions).  The combination must equal the
single-process oracle -- bitwise where §8(e) says so -- and each rank's
libjacc.so plan (built with world = 2 / 4) must have the counted copies of the
SURVEY count table.
"""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        res = {}
        # cfg2: histogram shards + allreduce(bins)  -> bitwise
        keys = synth.hist_keys(1 << 20, seed=7)
        lo, hi = synth.shard_range(keys.size, rank, world)
        bins = torch.from_numpy(oracle.histogram(keys[lo:hi], 256).astype(np.int64))
        dist.all_reduce(bins)
        res["hist"] = bool(np.array_equal(bins.numpy(), oracle.histogram(keys, 256)))
        # cfg1: vadd shard -> partial sum -> allreduce  (tolerance 1e-4 sum|x|)
        a, b = synth.vadd_inputs(1 << 16)
        lo, hi = synth.shard_range(a.size, rank, world)
        c = oracle.vadd(a[lo:hi], b[lo:hi])
        s = torch.tensor([oracle.reduce_sum(c)[0]], dtype=torch.float64)
        dist.all_reduce(s)
        ref, absum = oracle.reduce_sum(oracle.vadd(a, b))
        res["reduce"] = bool(abs(s.item() - ref) <= 1e-12 * absum)
        # cfg4: SGEMM row blocks (B replicated) + allgather rows -> bitwise
        A, B = synth.sgemm_inputs(64, 48, 80, "signed")
        lo, hi = synth.shard_range(64, rank, world)
        part = torch.from_numpy(oracle.sgemm_rows(A, B, np.arange(lo, hi)))
        parts = [torch.zeros((synth.shard_range(64, r, world)[1] - synth.shard_range(64, r, world)[0], 48),
                             dtype=torch.float64) for r in range(world)]
        dist.all_gather(parts, part)
        res["sgemm"] = bool(np.array_equal(torch.cat(parts).numpy(), oracle.sgemm_rows(A, B)))
        # cfg5: N-body target shards, positions all-gathered every step -> bitwise
        n, steps = 96, 3
        pos, vel = synth.nbody_state(n, seed=3)
        lo, hi = synth.shard_range(n, rank, world)
        P = pos.astype(np.float64).copy()
        V = vel[lo:hi].astype(np.float64).copy()
        for _ in range(steps):
            acc = oracle.nbody_accel(P, np.arange(lo, hi))
            V[:, :3] += acc * synth.NBODY_DT
            mine = P[lo:hi].copy()
            mine[:, :3] += V[:, :3] * synth.NBODY_DT
            gathered = [torch.zeros((synth.shard_range(n, r, world)[1] - synth.shard_range(n, r, world)[0], 4),
                                    dtype=torch.float64) for r in range(world)]
            dist.all_gather(gathered, torch.from_numpy(mine))
            P = torch.cat(gathered).numpy()
        fp, fv = oracle.nbody_steps(pos, vel, steps)
        res["nbody"] = bool(np.array_equal(P, fp) and np.array_equal(V, fv[lo:hi]))
        # f1: 2D convolution by row bands, r halo rows exchanged with the
        # neighbours (point-to-point, the NCCL path's ncclSend/ncclRecv),
        # then the band's rows of the convolution -> bitwise the full image's
        H, Wd, r = 61, 17, 2
        img = synth.uniform_f32(H * Wd, 95, -1, 1).reshape(H, Wd)
        f = synth.uniform_f32(25, 96, -1, 1).reshape(5, 5)
        blo, bhi = synth.shard_range(H, rank, world)
        band = torch.from_numpy(img[blo:bhi].copy())
        top = torch.zeros((r, Wd)); bot = torch.zeros((r, Wd))
        ops = []
        if rank > 0:
            ops += [dist.P2POp(dist.isend, band[:r].contiguous(), rank - 1),
                    dist.P2POp(dist.irecv, top, rank - 1)]
        if rank < world - 1:
            ops += [dist.P2POp(dist.isend, band[-r:].contiguous(), rank + 1),
                    dist.P2POp(dist.irecv, bot, rank + 1)]
        for w_ in dist.batch_isend_irecv(ops):
            w_.wait()
        ext = torch.cat([top, band, bot]).numpy()
        res["halo_ext"] = bool(np.array_equal(ext, oracle.halo_band(img, blo, bhi, r)))
        o, _ = oracle.conv2d(ext, f)
        res["conv_band"] = bool(np.array_equal(o[r:r + bhi - blo], oracle.conv2d(img, f)[0][blo:bhi]))
        # each rank's libjacc plan with world = 2: counted copies per rank
        import paper_1508_06791_b200 as J
        from paper_1508_06791_b200 import jacc
        g = J.Graph(rank=rank, world=world, nccl_comm=0x1)   # plan/dump only: NCCL is never called
        L = [np.zeros((n // world, 4), np.float32) for _ in range(2)]
        Vl = np.zeros((n // world, 4), np.float32)
        ALL = torch.zeros((n, 4), dtype=torch.float32)
        for k in range(10):
            g.add_task(J.JACC_OP_ALLGATHER, [g.a(L[k % 2], 1, True, f32x4=True),
                                             jacc.arg(ALL.data_ptr(), n, J.JACC_F32X4, 2, J.JACC_ARG_DEVICE)])
            g.add_task(J.JACC_OP_NBODY_STEP_F32, [jacc.arg(ALL.data_ptr(), n, J.JACC_F32X4, 1, J.JACC_ARG_DEVICE),
                                                   g.a(Vl, 3, True, f32x4=True), g.a(L[(k + 1) % 2], 2, True, f32x4=True)],
                       jacc.jacc_nbody_params_t(lo, 0.016, 0.01, 1.0))
        st = g.stats()
        res["plan"] = (st["h2d_count"], st["d2h_count"], st["collectives"], st["kernels"])
        g.destroy()
        # JACC_GRAPH_P2P (R23): the per-rank graphs of the same SPMD program
        # must agree on every collective's slot and on which collectives are
        # fused into their producers (the peer flags are matched by slot)
        g = J.Graph(rank=rank, world=world, flags=J.JACC_GRAPH_P2P)
        keys = np.zeros(1000 + rank, np.int32); bins = np.zeros(256, np.int32)
        s1 = np.zeros(1, np.float32)
        g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(keys, 1), g.a(bins, 2)], jacc.jacc_hist_params_t(256))
        g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(bins, 3)])
        g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(np.zeros(10 + rank, np.float32), 1), g.a(s1, 2)])
        g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(s1, 3)])
        for k in range(10):
            g.add_task(J.JACC_OP_ALLGATHER, [g.a(L[k % 2], 1, True, f32x4=True),
                                             jacc.arg(ALL.data_ptr(), n, J.JACC_F32X4, 2, J.JACC_ARG_DEVICE)])
            g.add_task(J.JACC_OP_NBODY_STEP_F32, [jacc.arg(ALL.data_ptr(), n, J.JACC_F32X4, 1, J.JACC_ARG_DEVICE),
                                                   g.a(Vl, 3, True, f32x4=True), g.a(L[(k + 1) % 2], 2, True, f32x4=True)],
                       jacc.jacc_nbody_params_t(lo, 0.016, 0.01, 1.0))
        fuse = [l for l in g.dump().splitlines() if l.startswith("fuse")]
        g.destroy()
        every = [None] * world
        dist.all_gather_object(every, fuse)
        res["p2p_fuse"] = (len(fuse), all(f == fuse for f in every))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, res))
    except Exception as e:   # surface the error to the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc()}))


@pytest.mark.parametrize("world", [2, 4])
def test_spmd_gloo(world):
    port = 29500 + (os.getpid() % 1000) + 7 * world
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in out[r], out[r].get("error")
        assert out[r]["hist"] and out[r]["reduce"] and out[r]["sgemm"] and out[r]["nbody"], out[r]
        assert out[r]["halo_ext"] and out[r]["conv_band"], out[r]
        assert out[r]["plan"] == (2, 3, 10, 10), out[r]["plan"]
        # hist+allreduce, reduce+allreduce, 9 nbody+allgather (the first allgather has no producer)
        assert out[r]["p2p_fuse"] == (11, True), out[r]["p2p_fuse"]


def test_shard_range_partition():
    import synth
    for n in (0, 1, 7, 1 << 20, 8192, 131072):
        for w in (1, 2, 3, 4, 8):
            rs = [synth.shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
