set -x
python -c "import torch; torch.zeros(1).cuda()"
for rep in 1 2; do
for db in 0 1; do for sh in 1 2 4 8; do JACC_NBODY_DB=$db timeout 300 python scripts/kbench.py nbody --shards $sh --reps 5 2>&1 | tail -1 | sed "s/^/db=$db sh=$sh /"; done; done
done
