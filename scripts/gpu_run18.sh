set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 600 python -m pytest tests -m gpu -q -x -k "graph or reduce or vadd" 2>&1 | tail -3
timeout 600 python -c "
import bench, torch, json
import paper_1508_06791_b200 as J
print(json.dumps(bench.cfg1_latency(torch, J)))
"
timeout 300 ncu --set full --clock-control none -k regex:unpack -c 1 -o gpurun_out/r18_unpack python scripts/kbench.py corr --reps 1 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/kbench.py corr --reps 1 2>/dev/null | grep -E "unpack|corr_i8" | cut -c1-200
