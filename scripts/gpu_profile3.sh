# Round-1 profile capture for the committed evidence (profiles/): launch list and DRAM traffic of the
# default bench step, ncu --set full of every hot kernel (plain and P2P-fused), bench JSON lines.
set -x
TAG=${TAG:-r1g}
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_traffic.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in nbody_partial nbody_finish gemm_3xtf32 hist256 bs_v4 vadd_v4 reduce_kernel split_bt split_a; do
  case $k in
    nbody*) op=nbody;; gemm*|split*) op=sgemm;; hist*) op=hist;; bs*) op=bs;; vadd*) op=vadd;; reduce*) op=reduce;;
  esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_full_$k python scripts/kbench.py $op --reps 1 > /dev/null 2>&1
done
for k in nbody_finish hist256 reduce_kernel; do
  case $k in nbody*) op=nbody;; hist*) op=hist;; reduce*) op=reduce;; esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_full_${k}_p2p python scripts/kbench.py $op --p2p --reps 1 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_p2p_launches.csv python scripts/kbench.py hist reduce nbody --p2p --reps 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_plain_launches.csv python scripts/kbench.py hist reduce nbody --reps 3 > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1
JACC_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29911 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_shared2.json 2> gpurun_out/${TAG}_bench_shared2.err
ls gpurun_out | grep $TAG
