set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -k "not 3xtf32" 2>&1 | tail -40 > gpurun_out/r1_pytest.txt
cat gpurun_out/r1_pytest.txt
timeout 300 python -m pytest tests -m gpu -q -x -k "3xtf32 and not full_size" 2>&1 | tail -40 > gpurun_out/r1_pytest_tf32.txt
cat gpurun_out/r1_pytest_tf32.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.txt 2>&1; tail -5 gpurun_out/r1_smoke.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err || \
  timeout 600 python bench.py --steps 5 --warmup 3 --sgemm-mode ffma > gpurun_out/r1_bench_ffma.json 2>> gpurun_out/r1_bench.err
tail -5 gpurun_out/r1_bench.err; cat gpurun_out/r1_bench*.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r1_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
wc -l gpurun_out/r1_launches.csv
