set -x
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -8
timeout 300 python scripts/kbench.py bs hist
timeout 900 python bench.py > gpurun_out/r5_bench.json 2> gpurun_out/r5_bench.err; tail -3 gpurun_out/r5_bench.err; cat gpurun_out/r5_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:bs_v4 -c 1 -o gpurun_out/r5_bs python scripts/kbench.py bs --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hist256 -c 1 -o gpurun_out/r5_hist python scripts/kbench.py hist --reps 1 > /dev/null 2>&1
