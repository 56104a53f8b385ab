set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "hist or nbody or graph or smoke" 2>&1 | tail -4
timeout 300 python scripts/kbench.py hist bs nbody
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r6_bench.json 2> gpurun_out/r6_bench.err; tail -3 gpurun_out/r6_bench.err; cat gpurun_out/r6_bench.json
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hist256 -c 1 -o gpurun_out/r6_hist python scripts/kbench.py hist --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:nbody_partial -c 1 -o gpurun_out/r6_nbody python scripts/kbench.py nbody --reps 1 > /dev/null 2>&1
