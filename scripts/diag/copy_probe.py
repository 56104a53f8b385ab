"""Host time of a 256 MiB pinned H2D cudaMemcpyAsync: torch copy_ vs the
runtime's execute (prepare_memory + issue)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1508_06791_b200 as J
from paper_1508_06791_b200.torch_glue import make_graph
big = 1 << 26
a = torch.empty(big, dtype=torch.float32).pin_memory().uniform_()
b = torch.empty(big, dtype=torch.float32).pin_memory().uniform_()
c = torch.empty(big, dtype=torch.float32).pin_memory()
d = torch.empty(big, device="cuda")
s = torch.cuda.Stream()
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        d.copy_(a, non_blocking=True)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("torch copy_ host %.3f ms, done %.3f ms" % ((t1 - t0) * 1e3, (t2 - t0) * 1e3), flush=True)
for i in range(3):
    g, st = make_graph(0)
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, 1), g.a(b, 1), g.a(c, 2)])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.execute()
    t1 = time.perf_counter()
    g.sync()
    t2 = time.perf_counter()
    g.execute()
    t3 = time.perf_counter()
    g.sync()
    t4 = time.perf_counter()
    print("jacc exec1 host %.3f ms (total %.3f); exec2 host %.3f ms (total %.3f)" % (
        (t1 - t0) * 1e3, (t2 - t0) * 1e3, (t3 - t2) * 1e3, (t4 - t2) * 1e3), flush=True)
    g.destroy()
