python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -c "
import json, torch, bench
import paper_1508_06791_b200 as J
torch.cuda.set_device(0)
print(json.dumps(bench.next_rows(torch, J, bench._peaks()), indent=1))
"
