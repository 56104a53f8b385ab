# Round-2 profile capture for profiles/: launch list and DRAM traffic of the default bench step,
# ncu --set full of every hot kernel (incl. the CTA-pair SGEMM and the paper-size HBM points).
set -x
TAG=${TAG:-r2}
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_traffic.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in nbody_partial nbody_finish gemm_3xtf32_pair hist256_w16 bs_v4 vadd_v4 reduce_kernel; do
  case $k in
    nbody*) op=nbody; n=0;; gemm*) op=sgemm; n=0;; hist*) op=hist; n=0;; bs*) op=bs; n=0;;
    vadd*) op=vadd; n=16777216;; reduce*) op=reduce; n=33554432;;
  esac
  # --no-flush: the L2 flush's torch.sum is a "reduce_kernel" too (ncu flushes caches itself)
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -o gpurun_out/${TAG}_full_$k python scripts/kbench.py $op --n $n --reps 1 --no-flush > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_3xtf32_pair -c 1 -o gpurun_out/${TAG}_full_gemm_rowblock8 python scripts/kbench.py sgemm --m 1024 --reps 1 > /dev/null 2>&1
ls gpurun_out | grep $TAG
