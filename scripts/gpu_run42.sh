# P2P tests, bench N=1 with plan replay, and the N=2 bench path with both ranks on the one GPU (P2P, gloo).
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_p2p.py tests/test_gpu_bench_suite.py -q -x 2>&1 | tail -5
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r42_bench.json 2> gpurun_out/r42_bench.err; tail -3 gpurun_out/r42_bench.err; cat gpurun_out/r42_bench.json
JACC_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r42_bench2.json 2> gpurun_out/r42_bench2.err; tail -20 gpurun_out/r42_bench2.err; cat gpurun_out/r42_bench2.json
