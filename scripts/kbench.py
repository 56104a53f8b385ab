#!/usr/bin/env python
"""Kernel micro-bench through the C-ABI (device-resident args), for timing a
single op in isolation and for short ncu captures:

    python scripts/kbench.py hist|bs|vadd|reduce|sgemm|nbody [--n N] [--reps R]

Prints one JSON line per op: mean/min device ms per launch (CUDA events on the
stream the task runs on = jacc_graph_task_ms) and achieved GB/s or TFLOP/s.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("ops", nargs="+")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--no-flush", action="store_true", help="no L2 flush between reps (warm L2 / back-to-back)")
    ap.add_argument("--mode", default="3xtf32")
    ap.add_argument("--m", type=int, default=0, help="sgemm: rows of A / C (default n; a 1/8 row block = 1024)")
    ap.add_argument("--shards", type=int, default=1, help="nbody: time rank 0's target shard of N/shards bodies")
    ap.add_argument("--p2p", action="store_true",
                    help="hist/reduce/nbody: follow the op with its collective (allreduce / allgather) in a "
                         "JACC_GRAPH_P2P graph at world 1, so the collective is fused into the op's kernel")
    a = ap.parse_args()
    import torch
    import paper_1508_06791_b200 as J
    from paper_1508_06791_b200 import jacc
    from paper_1508_06791_b200.torch_glue import make_graph, peer_tensor
    R, W, RW = J.JACC_READ, J.JACC_WRITE, J.JACC_READWRITE
    dev = torch.device("cuda", 0)
    from bench import L2Flush   # write + read flush: clean L2 lines (bench.py)
    flush = L2Flush(torch, dev)
    for op in a.ops:
        g, _ = make_graph(0, n_streams=1, flags=J.JACC_GRAPH_P2P if a.p2p else 0)
        keep = []

        def D(x):
            t = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
            keep.append(t)
            return t
        if op == "vadd":
            n = a.n or synth.CFG1_N
            x, y = synth.vadd_inputs(n)
            g.add_task(J.JACC_OP_VADD_F32, [g.a(D(x), R), g.a(D(y), R), g.a(D(np.zeros(n, np.float32)), W)])
            units, kind = 12 * n, "GB/s"
        elif op == "reduce":
            n = a.n or synth.CFG1_N
            out = D(np.zeros(1, np.float32))
            g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(D(synth.uniform_f32(n, 1)), R), g.a(out, W)])
            if a.p2p:
                g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(out, RW)])
            units, kind = 4 * n, "GB/s"
        elif op == "hist":
            n = a.n or synth.CFG2_N
            bins = D(np.zeros(256, np.int32))
            g.add_task(J.JACC_OP_HISTOGRAM_I32, [g.a(D(synth.hist_keys(n)), R), g.a(bins, W)],
                       jacc.jacc_hist_params_t(256))
            if a.p2p:
                g.add_task(J.JACC_OP_ALLREDUCE_SUM, [g.a(bins, RW)])
            units, kind = 4 * n, "GB/s"
        elif op == "bs":
            n = a.n or synth.CFG3_N
            g.add_task(J.JACC_OP_BLACKSCHOLES_F32, [g.a(D(synth.bs_rand(n)), R), g.a(D(np.zeros(n, np.float32)), W),
                                                     g.a(D(np.zeros(n, np.float32)), W)])
            units, kind = 12 * n, "GB/s"
        elif op == "sgemm":
            n = a.n or synth.CFG4_MNK
            m = a.m or n
            A, B = synth.sgemm_inputs(m, n, n)
            mode = J.JACC_SGEMM_3XTF32 if a.mode == "3xtf32" else J.JACC_SGEMM_FFMA
            g.add_task(J.JACC_OP_SGEMM_F32, [g.a(D(A), R), g.a(D(B), R), g.a(D(np.zeros((m, n), np.float32)), W)],
                       jacc.jacc_sgemm_params_t(m, n, n, n, n, n, mode, 0))
            units, kind = 2 * m * n * n, "TFLOP/s"
        elif op == "nbody":
            n = a.n or synth.CFG5_N
            pos, vel = synth.nbody_state(n)
            lo, hi = synth.shard_range(n, 0, a.shards)
            pout = D(np.zeros_like(pos[lo:hi]))
            g.add_task(J.JACC_OP_NBODY_STEP_F32, [g.a(D(pos), R, f32x4=True), g.a(D(vel[lo:hi]), RW, f32x4=True),
                                                   g.a(pout, W, f32x4=True)],
                       jacc.jacc_nbody_params_t(lo, synth.NBODY_DT, synth.NBODY_EPS2, synth.NBODY_G))
            if a.p2p:
                g.add_task(J.JACC_OP_ALLGATHER, [g.a(pout, R, f32x4=True), g.a(peer_tensor(g, (hi - lo, 4)), W, f32x4=True)])
            units, kind = 20 * n * (hi - lo), "TFLOP/s"
        elif op == "conv2d":
            n = a.n or 2048
            img = synth.uniform_f32(n * n, 11, -1, 1).reshape(n, n)
            f = synth.uniform_f32(25, 12, -1, 1).reshape(5, 5)
            g.add_task(J.JACC_OP_CONV2D_F32, [g.a(D(img), R), g.a(D(f), R), g.a(D(np.zeros_like(img)), W)],
                       jacc.jacc_conv2d_params_t(n, n, 2, 0))
            units, kind = 8 * n * n, "GB/s"
        elif op == "corr":
            A = synth.corr_bitsets(a.n) if a.n else synth.corr_bitsets()
            C = np.zeros((A.shape[0], A.shape[0]), np.int32)
            g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(D(A.view(np.int32)), R), g.a(D(A.view(np.int32) + 0), R),
                                                  g.a(D(C), W)],
                       jacc.jacc_corr_params_t(A.shape[0], A.shape[0], A.shape[1]))
            n = A.shape[0]
            units, kind = n * n * A.shape[1] * 32 * 2, "TFLOP/s"   # bit-ops: AND + count per bit pair
        elif op == "spmv":
            rp, col, val = synth.banded_csr(a.n, 23 * a.n) if a.n else synth.banded_csr()
            n = rp.size - 1
            x = synth.uniform_f32(n, 5, -1, 1)
            g.add_task(J.JACC_OP_SPMV_CSR_F32, [g.a(D(rp), R), g.a(D(col), R), g.a(D(val), R), g.a(D(x), R),
                                                 g.a(D(np.zeros(n, np.float32)), W)],
                       jacc.jacc_spmv_params_t(n, n))
            units, kind = 8 * col.size + 4 * (n + 1) + 8 * n, "GB/s"
        else:
            raise SystemExit(f"unknown op {op}")
        ms = []
        for i in range(a.reps + 2):
            if not a.no_flush:
                flush.fill_(1.0)
            torch.cuda.synchronize()
            g.run()
            if i >= 2:
                ms.append(g.task_ms(0))
        mean = sum(ms) / len(ms)
        scale = 1e9 if kind == "GB/s" else 1e12
        print(json.dumps({"op": op, "n": n, "mean_ms": mean, "min_ms": min(ms),
                          "achieved": units / (mean * 1e-3) / scale, "best": units / (min(ms) * 1e-3) / scale,
                          "unit": kind, "launches_per_task": g.stats()["launches"]}), flush=True)
        g.destroy()


if __name__ == "__main__":
    main()
