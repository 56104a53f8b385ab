# Full validation on a B200 (via gpurun): build, the GPU test suite, smoke(),
# the default bench, and the N = 2 bench path with both ranks time-sliced on
# the box's one GPU (JACC_BENCH_SHARED_GPU=1: exercises the multi-rank code,
# its numbers are not a measurement).
#   gpurun --timeout 3000 -- 'bash scripts/gpu_validate.sh'
set -x
TAG=${TAG:-val}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | cut -c1-120
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_bench.err
JACC_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 --steps 3 --warmup 3 \
  > gpurun_out/${TAG}_bench_shared2.json 2> gpurun_out/${TAG}_bench_shared2.err; tail -1 gpurun_out/${TAG}_bench_shared2.err
