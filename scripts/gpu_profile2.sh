# Round-1 (session 2) profile refresh: launch list of the default bench step, DRAM traffic per task,
# and P2P-fused vs plain kernels (world 1) side by side.
set -x
TAG=${TAG:-r1d}
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_traffic.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for op in hist reduce nbody; do
  for p in "" "--p2p"; do
    timeout 300 python scripts/kbench.py $op $p --reps 10 2>&1 | tail -1 | sed "s/^/kbench $p /"
  done
done
timeout 300 python scripts/kbench.py nbody --shards 8 --reps 10 2>&1 | tail -1 | sed "s/^/kbench sh8 /"
timeout 300 python scripts/kbench.py nbody --shards 8 --p2p --reps 10 2>&1 | tail -1 | sed "s/^/kbench sh8 --p2p /"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_p2p_launches.csv python scripts/kbench.py hist reduce nbody --p2p --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_plain_launches.csv python scripts/kbench.py hist reduce nbody --reps 3 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:nbody_finish -c 1 -o gpurun_out/${TAG}_full_nbody_finish_p2p python scripts/kbench.py nbody --shards 8 --p2p --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hist256 -c 1 -o gpurun_out/${TAG}_full_hist256_p2p python scripts/kbench.py hist --p2p --reps 1 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1
ls gpurun_out
