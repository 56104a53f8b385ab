#!/usr/bin/env python
"""profiles/traffic.json from an ncu metric capture of one bench step:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file gpurun_out/traffic.csv \
        python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline
    python scripts/ncu_traffic.py gpurun_out/traffic.csv > profiles/traffic.json

Per task (one jacc task = all CUDA kernels it launches) DRAM bytes read +
written, averaged over the task's instances in the capture.
"""
import csv
import json
import sys
from collections import defaultdict

TASK_OF = [("vadd_v4_kernel", "vadd"), ("vadd_v8_kernel", "vadd"), ("bs_v8_kernel", "bs"), ("jacc_k::<unnamed>::reduce_kernel", "reduce"), ("hist256", "hist"),
           ("bs_v4_kernel", "bs"), ("gemm_3xtf32_pair_kernel", "sgemm"), ("split_a_kernel", "sgemm"),
           ("split_bt_kernel", "sgemm"), ("gemm_3xtf32_kernel", "sgemm"), ("nbody_partial", "nbody"),
           ("nbody_finish_kernel", "nbody")]


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = defaultdict(lambda: defaultdict(float))
    launches = defaultdict(lambda: defaultdict(set))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        for pat, task in TASK_OF:
            if pat in r[ki]:
                if r[mi].startswith("dram__bytes"):
                    per[task]["bytes"] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
                launches[task][pat].add(r[0])
    out = {"_source": f"{path}: ncu dram__bytes_read.sum + dram__bytes_write.sum per kernel, summed over the "
                      "kernels of a task, divided by the task's instances in one bench step"}
    for task, d in per.items():
        # a task's instances: launches of its most frequent kernel (N-body: 10 partial + 10 finish = 10 steps)
        n = max((len(v) for v in launches[task].values()), default=0) or 1
        out[task] = {"bytes_per_task": d["bytes"] / n, "instances": n}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
