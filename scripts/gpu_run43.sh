# Runtime issue overheads (plan cache, dep events on demand, NO_TIMING, reduce assign, triple merge): tests + cfg1 latency.
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -8
timeout 600 python -c "
import json, torch, bench
import paper_1508_06791_b200 as J
torch.cuda.set_device(0)
print(json.dumps(bench.cfg1_latency(torch, J), indent=1))
"
