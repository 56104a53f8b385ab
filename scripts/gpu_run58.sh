python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_next.py -q -x 2>&1 | tail -2
for n in 0 4096 8192; do timeout 300 python scripts/kbench.py corr --n $n --reps 10 2>&1 | tail -1 | cut -c1-120; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r58_corr.csv python scripts/kbench.py corr --reps 2 > /dev/null 2>&1
