# LL small allreduce + acq_rel fences: P2P tests and fused-vs-plain kernel times.
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_graph.py -q -x 2>&1 | tail -3
for op in hist reduce; do
  for p in "" "--p2p"; do timeout 300 python scripts/kbench.py $op $p --reps 20 2>&1 | tail -1 | sed "s/^/kbench $p /"; done
done
for p in "" "--p2p"; do timeout 300 python scripts/kbench.py nbody --shards 8 $p --reps 20 2>&1 | tail -1 | sed "s/^/kbench sh8 $p /"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r44_p2p_launches.csv python scripts/kbench.py hist reduce nbody --p2p --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r44_plain_launches.csv python scripts/kbench.py hist reduce nbody --reps 3 > /dev/null 2>&1
