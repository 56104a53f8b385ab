set -x
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/r2_pytest.txt; cat gpurun_out/r2_pytest.txt
timeout 300 python scripts/kbench.py vadd reduce hist bs sgemm nbody > gpurun_out/r2_kbench.txt 2>&1; cat gpurun_out/r2_kbench.txt
JACC_NBODY_VARIANT=s timeout 300 python scripts/kbench.py nbody > gpurun_out/r2_kbench_nbody_scalar.txt 2>&1; cat gpurun_out/r2_kbench_nbody_scalar.txt
timeout 300 ncu --set full --import-source on -k regex:nbody_partial -c 1 -o gpurun_out/r2_nbody_x2 python scripts/kbench.py nbody --reps 1 > /dev/null 2>&1
JACC_NBODY_VARIANT=s timeout 300 ncu --set full --import-source on -k regex:nbody_partial -c 1 -o gpurun_out/r2_nbody_s python scripts/kbench.py nbody --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:bs_v4 -c 1 -o gpurun_out/r2_bs python scripts/kbench.py bs --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:hist256 -c 1 -o gpurun_out/r2_hist python scripts/kbench.py hist --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on -k regex:gemm_3xtf32 -c 1 -o gpurun_out/r2_gemm python scripts/kbench.py sgemm --reps 1 > /dev/null 2>&1
ls -la gpurun_out/
