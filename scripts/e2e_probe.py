"""Where does the host-buffer cfg1 graph spend its time?  Splits execute /
sync host time, per-task device ms, and compares with the bare torch copy
sequence.  python scripts/e2e_probe.py"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1508_06791_b200 as J  # noqa: E402
from paper_1508_06791_b200.torch_glue import make_graph  # noqa: E402

R, W = J.JACC_READ, J.JACC_WRITE
a, b = synth.vadd_inputs()
ta, tb = torch.from_numpy(a).pin_memory(), torch.from_numpy(b).pin_memory()
tc, ts = torch.empty(a.size, pin_memory=True), torch.empty(1, pin_memory=True)
print("pinned", ta.is_pinned(), tb.is_pinned(), tc.is_pinned(), ts.is_pinned())
out = {}
for name, ns, flags in (("s2", 2, 0), ("s1", 1, 0), ("serial", 1, J.JACC_GRAPH_SERIAL), ("merge", 2, J.JACC_GRAPH_MERGE)):
    g, strm = make_graph(0, n_streams=ns, flags=flags)
    g.add_task(J.JACC_OP_VADD_F32, [g.a(ta, R), g.a(tb, R), g.a(tc, W)])
    g.add_task(J.JACC_OP_REDUCE_SUM_F32, [g.a(tc, R), g.a(ts, W)])
    for _ in range(5):
        g.run()
    te = ts_ = 0.0
    reps = 50
    for _ in range(reps):
        t0 = time.perf_counter(); g.execute(); t1 = time.perf_counter(); g.sync(); t2 = time.perf_counter()
        te += t1 - t0; ts_ += t2 - t1
    # device timeline of one execute: events on the graph's own streams
    ev = {k: torch.cuda.Event(enable_timing=True) for k in ("start", "h2d", "comp", "d2h")}
    torch.cuda.synchronize()
    ev["start"].record(strm["h2d"])
    g.execute()
    ev["h2d"].record(strm["h2d"])
    ev["comp"].record(strm["compute"][0])
    ev["d2h"].record(strm["d2h"])
    g.sync()
    torch.cuda.synchronize()
    timeline = {k: ev["start"].elapsed_time(ev[k]) * 1e3 for k in ("h2d", "comp", "d2h")}
    out[name] = {"execute_us": te / reps * 1e6, "sync_us": ts_ / reps * 1e6, "timeline_us": timeline,
                 "task_ms": [g.task_ms(0), g.task_ms(1)], "stats": {k: v for k, v in g.stats().items() if not k.startswith("total")}}
    g.destroy()
# bare torch: same copies + kernels
da, db = torch.empty_like(ta, device="cuda"), torch.empty_like(tb, device="cuda")
s = torch.cuda.Stream()
for _ in range(5):
    with torch.cuda.stream(s):
        da.copy_(ta, non_blocking=True); db.copy_(tb, non_blocking=True)
        dc = da + db; dsum = dc.sum()
        tc.copy_(dc, non_blocking=True); ts.copy_(dsum.view(1), non_blocking=True)
    s.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    with torch.cuda.stream(s):
        da.copy_(ta, non_blocking=True); db.copy_(tb, non_blocking=True)
        dc = da + db; dsum = dc.sum()
        tc.copy_(dc, non_blocking=True); ts.copy_(dsum.view(1), non_blocking=True)
    s.synchronize()
out["torch_one_stream_us"] = (time.perf_counter() - t0) / 50 * 1e6
print(json.dumps(out, indent=1))
