set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "bs or schedule or smoke" 2>&1 | tail -4
timeout 300 python scripts/kbench.py bs --reps 20
JACC_BS_V4=1 timeout 300 python scripts/kbench.py bs --reps 20
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_tma -c 1 -o gpurun_out/r12_bs_tma python scripts/kbench.py bs --reps 1 > /dev/null 2>&1
