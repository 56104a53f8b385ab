python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_next.py -q -x 2>&1 | grep -E "^E |FAILED|passed|failed" | head -12
