# Session re-entry validation: full GPU test suite, smoke, default bench.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r40_pytest.txt; cat gpurun_out/r40_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r40_smoke.txt 2>&1; tail -3 gpurun_out/r40_smoke.txt
timeout 900 python bench.py > gpurun_out/r40_bench.json 2> gpurun_out/r40_bench.err; tail -3 gpurun_out/r40_bench.err; cat gpurun_out/r40_bench.json
