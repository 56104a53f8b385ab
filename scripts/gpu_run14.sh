set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "sgemm or hist or smoke" 2>&1 | tail -4
timeout 300 python scripts/kbench.py sgemm hist --reps 10
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_3xtf32 -c 1 python scripts/kbench.py sgemm --reps 1 2>&1 | grep -E "dram__|duration|tensor"
