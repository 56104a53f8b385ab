set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "sgemm_gates or graph or nbody" 2>&1 | tail -4
timeout 300 python scripts/kbench.py sgemm
for v in "4,0" "4,1" "3,1" "5,1" "5,2" "2,0"; do JACC_NBODY_VARIANT=$v timeout 120 python scripts/kbench.py nbody --reps 4 | sed "s/^/$v /"; done
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:gemm_3xtf32 -c 1 python scripts/kbench.py sgemm --reps 1 2>&1 | grep -E "dram__|duration|tensor"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r8_bench.json 2> gpurun_out/r8_bench.err; tail -3 gpurun_out/r8_bench.err; python -c "import json;d=json.load(open('gpurun_out/r8_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['ms_per_step'],d.get('cfg1_task_graph'))"
