set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "sgemm or nbody" 2>&1 | tail -5
for v in "2,0" "0,4" "2,2" "2,1" "3,2" "1,2" "1,1"; do JACC_NBODY_VARIANT=$v timeout 120 python scripts/kbench.py nbody --reps 5 | sed "s/^/$v /"; done
timeout 300 python scripts/kbench.py bs hist sgemm
timeout 300 ncu --set full --clock-control none --import-source on -k regex:nbody_partial -c 1 -o gpurun_out/r3_nbody22 python scripts/kbench.py nbody --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_v4 -c 1 -o gpurun_out/r3_bs python scripts/kbench.py bs --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hist256 -c 1 -o gpurun_out/r3_hist python scripts/kbench.py hist --reps 1 > /dev/null 2>&1
