set -x
python -c "import torch; torch.zeros(1).cuda()"   # page in torch/CUDA once
for v in "3 4" "4 4" "2 4" "3 8" "2 8" "3 2" "4 2" "2 16"; do set -- $v; JACC_NBODY_PAIRS=$1 JACC_NBODY_UNROLL=$2 timeout 300 python scripts/kbench.py nbody --reps 4 | sed "s/^/P=$1 U=$2 /"; done
timeout 600 python -m pytest tests -m gpu -q -x -k "sgemm_gates or nbody" 2>&1 | tail -3
timeout 300 python scripts/kbench.py sgemm --reps 10
