"""Diagnose out-of-order issue: does a device-input task wait for an
unrelated task's large H2D?  Prints event times per phase."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1508_06791_b200 as J
from paper_1508_06791_b200.torch_glue import make_graph
R, W = 1, 2
big = 1 << 26
a = torch.empty(big, dtype=torch.float32).pin_memory().uniform_()
b = torch.empty(big, dtype=torch.float32).pin_memory().uniform_()
c = torch.empty(big, dtype=torch.float32).pin_memory()
print("pinned", a.is_pinned(), b.is_pinned(), c.is_pinned())
x = torch.rand(1 << 20, device="cuda"); y = torch.rand(1 << 20, device="cuda")
z = torch.empty(1 << 20, device="cuda")
for trial in range(3):
    g, st = make_graph(0)
    g.add_task(J.JACC_OP_VADD_F32, [g.a(a, R), g.a(b, R), g.a(c, W)])
    g.add_task(J.JACC_OP_VADD_F32, [g.a(x, R), g.a(y, R), g.a(z, W)])
    streams = [int(l.split("stream=")[1].split()[0]) for l in g.dump().splitlines() if l.startswith("task")]
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_start.record(st["h2d"])
    h0 = time.perf_counter()
    g.execute()
    h1 = time.perf_counter()
    e_t1 = torch.cuda.Event(enable_timing=True); e_t1.record(st["compute"][streams[1]])
    e_h2d = torch.cuda.Event(enable_timing=True); e_h2d.record(st["h2d"])
    g.sync()
    torch.cuda.synchronize()
    print(trial, "streams", streams, "host execute ms %.3f" % ((h1 - h0) * 1e3),
          "t1 done %.3f" % t_start.elapsed_time(e_t1), "h2d done %.3f" % t_start.elapsed_time(e_h2d),
          "t1 task_ms %.3f" % g.task_ms(1))
    g.destroy()
