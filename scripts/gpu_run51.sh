set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_next.py -q -x 2>&1 | tail -3
for n in 2048 8192 16384; do timeout 300 python scripts/kbench.py conv2d --n $n --reps 10 2>&1 | tail -1; done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv -c 1 -o gpurun_out/r51_full_conv python scripts/kbench.py conv2d --n 16384 --reps 1 > /dev/null 2>&1
