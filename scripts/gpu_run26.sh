set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
TAG=r1c bash scripts/gpu_profile.sh
