# Full validation of the current tree.
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1 | cut -c1-80
/usr/bin/time -f "bench wall %e s" timeout 1200 python bench.py > gpurun_out/r59_bench.json 2> gpurun_out/r59_bench.err; tail -2 gpurun_out/r59_bench.err
JACC_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/r59_bench_shared2.json 2> gpurun_out/r59_bench_shared2.err; tail -1 gpurun_out/r59_bench_shared2.err
