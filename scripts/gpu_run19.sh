set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 600 python -m pytest tests -m gpu -q -x -k "bs or schedule or smoke" 2>&1 | tail -3
timeout 300 python scripts/kbench.py bs --reps 20
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_v4 -c 1 -o gpurun_out/r19_bs python scripts/kbench.py bs --reps 1 > /dev/null 2>&1
