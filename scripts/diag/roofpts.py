"""bench.roofline_points alone (vadd 2^24, reduce 2^25, both 2^28): isolated
and back-to-back per-launch times."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_1508_06791_b200 as J
print(json.dumps(bench.roofline_points(torch, J, bench._peaks()), indent=1))
