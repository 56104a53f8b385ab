set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "graph or next or nbody or smoke" 2>&1 | tail -4
timeout 300 python scripts/kbench.py conv2d nbody
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r9_bench.json 2> gpurun_out/r9_bench.err; tail -3 gpurun_out/r9_bench.err; python -c "import json;d=json.load(open('gpurun_out/r9_bench.json'));print(d['value'],d['ms_per_step'],d['e2e']['ms_per_step'],d.get('cfg1_task_graph'))"
