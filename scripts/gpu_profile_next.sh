# ncu evidence for the §8(f) NEXT-row kernels (profiles/r1_ncu_next_rows.md):
# launch lists of scripts/kbench.py and one --set full capture per kernel.
#   gpurun --timeout 1500 -- 'TAG=r1n bash scripts/gpu_profile_next.sh'
set -x
TAG=${TAG:-r1n}
python -c "import __graft_entry__ as g; g.build()" > /dev/null
L="ncu --metrics gpu__time_duration.sum --clock-control none --csv"
timeout 600 $L --log-file gpurun_out/${TAG}_next_launches.csv sh -c \
  'python scripts/kbench.py conv2d --n 16384 --reps 3; python scripts/kbench.py conv2d --n 2048 --reps 3; python scripts/kbench.py spmv --n 2097152 --reps 3; python scripts/kbench.py corr --reps 3' > /dev/null 2>&1
F="ncu --set full --clock-control none --import-source on -c 1"
timeout 300 $F -k regex:conv2d_tma -o gpurun_out/${TAG}_full_conv2d_tma python scripts/kbench.py conv2d --n 16384 --reps 1 > /dev/null 2>&1
timeout 300 $F -k regex:conv2d_tma -o gpurun_out/${TAG}_full_conv2d_tma_2048 python scripts/kbench.py conv2d --n 2048 --reps 1 > /dev/null 2>&1
timeout 300 $F -k regex:spmv -o gpurun_out/${TAG}_full_spmv python scripts/kbench.py spmv --n 2097152 --reps 1 > /dev/null 2>&1
timeout 300 $F -k regex:corr_i8 -o gpurun_out/${TAG}_full_corr_i8 python scripts/kbench.py corr --reps 1 > /dev/null 2>&1
timeout 300 $F -k regex:unpack -o gpurun_out/${TAG}_full_corr_unpack python scripts/kbench.py corr --reps 1 > /dev/null 2>&1
ls gpurun_out | grep $TAG
