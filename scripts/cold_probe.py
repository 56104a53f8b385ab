"""Where does the first execute of a fresh cfg1 graph spend its time?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1508_06791_b200 as J
from paper_1508_06791_b200.torch_glue import make_graph
torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
a, b = synth.vadd_inputs()
for trial in range(3):
    ta, tb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
    tc, ts = torch.empty(a.size, pin_memory=True), torch.empty(1, pin_memory=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g, _ = make_graph(0, n_streams=2, flags=J.JACC_GRAPH_MERGE)
    t1 = time.perf_counter()
    g.add_task(J.JACC_OP_VADD_F32, [g.a(ta, 1, True), g.a(tb, 1, True), g.a(tc, 2)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(tc, 1), g.a(ts, 2)])
    t2 = time.perf_counter()
    g.execute()
    t3 = time.perf_counter()
    g.sync()
    t4 = time.perf_counter()
    g.run()
    t5 = time.perf_counter()
    print(f"trial {trial}: make_graph {1e6*(t1-t0):.0f} us, add {1e6*(t2-t1):.0f} us, execute {1e6*(t3-t2):.0f} us, "
          f"sync {1e6*(t4-t3):.0f} us, second run {1e6*(t5-t4):.0f} us", flush=True)
    g.destroy()
    if trial == 0:
        torch.cuda.empty_cache()
