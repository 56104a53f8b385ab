set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 600 python -m pytest tests -m gpu -q -x -k "nbody" 2>&1 | tail -3
for sh in 1 2 8; do timeout 300 python scripts/kbench.py nbody --shards $sh --reps 5 2>&1 | tail -1; done
