python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_bench_suite.py -q -x -k world2 2>&1 | grep -E "Error|error|assert|Traceback|File" | head -30
