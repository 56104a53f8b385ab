# P2P collectives: world-1 and two-process world-2 on the one GPU; full GPU suite for regressions.
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_p2p.py -q -x 2>&1 | tail -30 > gpurun_out/r41_p2p.txt; cat gpurun_out/r41_p2p.txt
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/r41_pytest.txt; cat gpurun_out/r41_pytest.txt
