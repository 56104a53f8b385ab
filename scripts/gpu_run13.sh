set -x
timeout 300 python -m pytest tests -m gpu -q -x -k "hist" 2>&1 | tail -3
timeout 300 python scripts/kbench.py hist --reps 20
JACC_HIST_ATOM=1 timeout 300 python scripts/kbench.py hist --reps 20
JACC_HIST_ATOM=1 timeout 300 python -m pytest tests -m gpu -q -x -k "hist" 2>&1 | tail -3
