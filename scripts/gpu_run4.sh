set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "hist or bs or graph or nbody" 2>&1 | tail -5
for v in "2,0" "3,0" "4,0" "1,0"; do JACC_NBODY_VARIANT=$v timeout 120 python scripts/kbench.py nbody --reps 5 | sed "s/^/$v /"; done
timeout 300 python scripts/kbench.py bs hist vadd reduce
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r4_bench.json 2> gpurun_out/r4_bench.err; tail -3 gpurun_out/r4_bench.err; cat gpurun_out/r4_bench.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_v4 -c 1 -o gpurun_out/r4_bs python scripts/kbench.py bs --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hist256 -c 1 -o gpurun_out/r4_hist python scripts/kbench.py hist --reps 1 > /dev/null 2>&1
