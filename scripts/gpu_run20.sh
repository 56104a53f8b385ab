set -x
python -c "import torch; torch.zeros(1).cuda()"
for v in 0 1 2 3; do JACC_BS_VARIANT=$v timeout 300 python scripts/kbench.py bs --reps 20 | sed "s/^/v$v /"; done
