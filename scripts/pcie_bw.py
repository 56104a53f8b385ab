"""Host<->device copy bandwidth from pinned memory (cudaMemcpyAsync via
torch), for reading the e2e numbers: python scripts/pcie_bw.py"""
import json

import torch

out = {}
for mib in (4, 8, 64, 256):
    n = mib << 18
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out["%s_%dMiB" % (name, mib)] = {"us": round(ms * 1e3, 1), "GB/s": round(n * 4 / ms / 1e6, 1)}
print(json.dumps(out))
