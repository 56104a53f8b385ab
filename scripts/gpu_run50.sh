# NEXT rows (f1 conv2d, f3 corr, f4 SpMV): paper sizes and roofline-point sizes, + ncu of each kernel.
set -x
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for n in 2048 8192 16384; do timeout 300 python scripts/kbench.py conv2d --n $n --reps 10 2>&1 | tail -1; done
for n in 0 4096 8192; do timeout 300 python scripts/kbench.py corr --n $n --reps 10 2>&1 | tail -1; done
for n in 0 4194304; do timeout 600 python scripts/kbench.py spmv --n $n --reps 10 2>&1 | tail -1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r50_next_launches.csv python scripts/kbench.py conv2d corr spmv --reps 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv -c 1 -o gpurun_out/r50_full_conv python scripts/kbench.py conv2d --n 16384 --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:corr -c 2 -o gpurun_out/r50_full_corr python scripts/kbench.py corr --reps 1 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:unpack -c 1 -o gpurun_out/r50_full_unpack python scripts/kbench.py corr --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv -c 1 -o gpurun_out/r50_full_spmv python scripts/kbench.py spmv --n 4194304 --reps 1 > /dev/null 2>&1
ls gpurun_out | grep r50
