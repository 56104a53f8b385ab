set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for sh in 1 2 4 8; do timeout 300 python scripts/kbench.py nbody --shards $sh --reps 5 2>&1 | tail -1; done
timeout 900 python bench.py > gpurun_out/r31_bench.json 2> gpurun_out/r31_bench.err; tail -3 gpurun_out/r31_bench.err; cat gpurun_out/r31_bench.json
