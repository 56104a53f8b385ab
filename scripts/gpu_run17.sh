set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python scripts/kbench.py corr nbody sgemm --reps 10
timeout 900 python bench.py > gpurun_out/r17_bench.json 2> gpurun_out/r17_bench.err; tail -3 gpurun_out/r17_bench.err; python -c "import json;d=json.load(open('gpurun_out/r17_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['ms_per_step'],d['roofline'],d['clocks'])"
