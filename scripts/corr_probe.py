# corr time vs. problem size (device time per call, L2 flushed): python scripts/corr_probe.py [terms] [docs]
import sys, json, numpy as np, torch
sys.path.insert(0, ".")
import synth
import paper_1508_06791_b200 as J
from paper_1508_06791_b200 import jacc
from paper_1508_06791_b200.torch_glue import make_graph
R, W = J.JACC_READ, J.JACC_WRITE
dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, device=dev)
TERMS = [int(a) for a in sys.argv[1:2]] or [1024, 2048]
DOCS = [int(a) for a in sys.argv[2:3]] or [4096, 8192, 16384, 32768, 65536, 131072]
for terms in TERMS:
    for docs in DOCS:
        bits = synth.corr_bitsets(terms, docs)
        A = torch.from_numpy(bits.view(np.int32)).to(dev)
        C = torch.empty((terms, terms), dtype=torch.int32, device=dev)
        g, _ = make_graph(0, n_streams=1)
        g.add_task(J.JACC_OP_CORR_POPC_U32, [g.a(A, R), g.a(A, R), g.a(C, W)], jacc.jacc_corr_params_t(terms, terms, docs // 32))
        ms = []
        for i in range(12):
            flush.fill_(1.0); torch.cuda.synchronize(); g.run()
            if i >= 2: ms.append(g.task_ms(0))
        g.destroy()
        ops = 2 * terms * terms * docs
        print(json.dumps({"terms": terms, "docs": docs, "us": round(1e3 * float(np.mean(ms)), 2), "tops": round(ops / (np.mean(ms) * 1e-3) / 1e12, 1)}), flush=True)
