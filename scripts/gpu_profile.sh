# Round profile capture: launch list + traffic + full captures of every hot kernel.
set -x
TAG=${TAG:-r1}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_traffic.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in nbody_partial gemm_3xtf32 hist256 bs_v4 vadd_v4 reduce_kernel split_bt split_a; do
  case $k in
    nbody*) op=nbody;; gemm*|split*) op=sgemm;; hist*) op=hist;; bs*) op=bs;; vadd*) op=vadd;; reduce*) op=reduce;;
  esac
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_full_$k python scripts/kbench.py $op --reps 1 > /dev/null 2>&1
done
ls gpurun_out
