set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for op in hist reduce; do for p in "" "--p2p"; do timeout 300 python scripts/kbench.py $op $p --reps 20 2>&1 | tail -1 | sed "s/^/$op $p /"; done; done
for sh in 1 8; do for p in "" "--p2p"; do timeout 300 python scripts/kbench.py nbody --shards $sh $p --reps 10 2>&1 | tail -1 | sed "s/^/nbody sh$sh $p /"; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r46_p2p_launches.csv python scripts/kbench.py hist reduce nbody --p2p --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r46_plain_launches.csv python scripts/kbench.py hist reduce nbody --reps 3 > /dev/null 2>&1
