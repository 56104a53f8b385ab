set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_bench_suite.py -q -x 2>&1 | tail -3
timeout 300 python scripts/cold_probe.py
