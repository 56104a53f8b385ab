set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 300 python scripts/e2e_probe.py
for c in 1024 1536 2048 2560 3072; do JACC_NBODY_VAR=0 JACC_NBODY_CHUNK=$c timeout 300 python scripts/kbench.py nbody --reps 5 2>&1 | tail -1; done
for v in 3 5; do JACC_NBODY_VAR=$v JACC_NBODY_CHUNK=2048 timeout 300 python scripts/kbench.py nbody --reps 5 2>&1 | tail -1; done
for c in 2048 1024; do JACC_NBODY_VAR=0 JACC_NBODY_CHUNK=$c timeout 300 python scripts/kbench.py nbody --n 16384 --reps 20 2>&1 | tail -1; done
JACC_NBODY_VAR=0 JACC_NBODY_CHUNK=8192 timeout 300 python scripts/kbench.py nbody --n 16384 --reps 20 2>&1 | tail -1
