set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "schedule or next" 2>&1 | tail -4
bash scripts/gpu_sanitize.sh
