set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_bench_suite.py -q -x 2>&1 | tail -3
JACC_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r48_bench_shared2.json 2> gpurun_out/r48_bench_shared2.err; tail -3 gpurun_out/r48_bench_shared2.err
