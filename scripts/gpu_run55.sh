python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_next.py -q -x 2>&1 | tail -1
for n in 0 4194304; do timeout 600 python scripts/kbench.py spmv --n $n --reps 10 2>&1 | tail -1 | cut -c1-140; done
