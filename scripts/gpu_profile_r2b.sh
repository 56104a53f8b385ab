# Final round-2 profile capture for profiles/ (tag r2b): launch list and DRAM
# traffic of the default bench step, ncu --set full of the hot kernels as they
# now stand (incl. the 256-bit Black-Scholes and vadd kernels and the 16-bit
# split-K corr epilogue), the NEXT-row kernels, the bench JSON lines (own arm,
# reference arm, the N = 2 path on one GPU) and the sanitizer pass.
#   gpurun --timeout 3600 -- 'bash scripts/gpu_profile_r2b.sh'
set -x
TAG=${TAG:-r2b}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
L="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
F="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $L --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_traffic.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for k in nbody_partial nbody_finish gemm_3xtf32_pair hist256_w16 bs_v8; do
  case $k in nbody*) op=nbody;; gemm*) op=sgemm;; hist*) op=hist;; bs*) op=bs;; esac
  timeout 300 $F -k regex:$k -o gpurun_out/${TAG}_full_$k python scripts/kbench.py $op --reps 1 --no-flush > /dev/null 2>&1
done
timeout 300 $F -k regex:vadd_v4 -o gpurun_out/${TAG}_full_vadd_v4_2p24 python scripts/kbench.py vadd --n 16777216 --reps 1 --no-flush > /dev/null 2>&1
timeout 300 $F -k regex:vadd_v8 -o gpurun_out/${TAG}_full_vadd_v8_2p28 python scripts/kbench.py vadd --n 268435456 --reps 1 --no-flush > /dev/null 2>&1
timeout 300 $F -k regex:reduce_kernel -o gpurun_out/${TAG}_full_reduce_2p25 python scripts/kbench.py reduce --n 33554432 --reps 1 --no-flush > /dev/null 2>&1
timeout 300 $F -k regex:gemm_3xtf32_pair -o gpurun_out/${TAG}_full_gemm_rowblock8 python scripts/kbench.py sgemm --m 1024 --reps 1 > /dev/null 2>&1
timeout 600 $L --log-file gpurun_out/${TAG}_next_launches.csv sh -c \
  'python scripts/kbench.py conv2d --n 16384 --reps 3; python scripts/kbench.py conv2d --n 2048 --reps 3; python scripts/kbench.py spmv --n 2097152 --reps 3; python scripts/kbench.py corr --reps 3' > /dev/null 2>&1
timeout 300 $F -k regex:corr_i8 -o gpurun_out/${TAG}_full_corr_i8 python scripts/kbench.py corr --reps 1 > /dev/null 2>&1
timeout 300 $F -k regex:spmv -o gpurun_out/${TAG}_full_spmv python scripts/kbench.py spmv --n 2097152 --reps 1 > /dev/null 2>&1
timeout 300 $F -k regex:conv2d_tma -o gpurun_out/${TAG}_full_conv2d_tma python scripts/kbench.py conv2d --n 16384 --reps 1 > /dev/null 2>&1
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; tail -2 gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
JACC_BENCH_SHARED_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_shared2.json 2> gpurun_out/${TAG}_bench_shared2.err
timeout 1800 bash scripts/gpu_sanitize.sh > gpurun_out/${TAG}_sanitize.txt 2>&1
ls gpurun_out | grep $TAG
