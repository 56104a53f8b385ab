set -x
python -c "import torch; torch.zeros(1).cuda()"
python scripts/pcie_bw.py
for v in 0 1 2 3 4 5; do JACC_NBODY_VAR=$v timeout 300 python scripts/kbench.py nbody --reps 5 2>&1 | tail -1; done
for c in 4352 5632 7936 1536; do JACC_NBODY_VAR=2 JACC_NBODY_CHUNK=$c timeout 300 python scripts/kbench.py nbody --reps 5 2>&1 | tail -1; done
for c in 7424 4352 2048; do JACC_NBODY_VAR=0 JACC_NBODY_CHUNK=$c timeout 300 python scripts/kbench.py nbody --reps 5 2>&1 | tail -1; done
for pf in 0 2 4 8 0; do JACC_HIST_PF=$pf timeout 300 python scripts/kbench.py hist --reps 20 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_graph.py -q 2>&1 | tail -3
