python -c "import __graft_entry__ as g; g.build()" > /dev/null
t0=$(date +%s); timeout 1200 python bench.py > gpurun_out/r60_bench.json 2> gpurun_out/r60_bench.err; echo "bench wall $(( $(date +%s) - t0 )) s"; tail -2 gpurun_out/r60_bench.err
