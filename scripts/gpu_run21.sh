set -x
python -c "import torch; torch.zeros(1).cuda()"
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r21_bench.json 2> gpurun_out/r21_bench.err; tail -3 gpurun_out/r21_bench.err; cat gpurun_out/r21_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r21_ref.json 2>&1; tail -2 gpurun_out/r21_ref.json
TAG=r1b bash scripts/gpu_profile.sh
