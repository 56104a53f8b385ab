set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "next or graph" 2>&1 | tail -4
timeout 300 python scripts/kbench.py conv2d corr spmv
timeout 600 python -c "
import bench, torch, json
import paper_1508_06791_b200 as J
print(json.dumps(bench.cfg1_latency(torch, J)))
"
