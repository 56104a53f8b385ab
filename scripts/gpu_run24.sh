set -x
python -c "import torch; torch.zeros(1).cuda()"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_pipes scripts/micro/fp32_pipes.cu && timeout 120 /tmp/fp32_pipes
timeout 300 python scripts/e2e_probe.py
for sh in 1 2 4 8; do timeout 300 python scripts/kbench.py nbody --shards $sh --reps 5 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -q -k "nbody" 2>&1 | tail -3
