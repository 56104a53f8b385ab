set -x
python -c "import __graft_entry__ as g; g.build()"
for op in hist reduce; do timeout 300 python scripts/kbench.py $op --p2p --reps 20 2>&1 | tail -1 | sed "s/^/kbench $p /"; done
for x in 0 1 2 3; do JACC_EXP=$x timeout 300 python scripts/kbench.py nbody --p2p --reps 10 2>&1 | tail -1 | sed "s/^/exp$x full /"; done
for x in 0 1 2 3; do JACC_EXP=$x timeout 300 python scripts/kbench.py nbody --shards 8 --p2p --reps 20 2>&1 | tail -1 | sed "s/^/exp$x sh8 /"; done
timeout 300 python scripts/kbench.py nbody --reps 10 2>&1 | tail -1 | sed "s/^/plain full /"
