python -c "import __graft_entry__ as g; g.build()" > /dev/null
for e in 1 5 6; do for n in 0 4194304; do JACC_SPMV=$e timeout 600 python scripts/kbench.py spmv --n $n --reps 10 2>&1 | tail -1 | cut -c1-70 | sed "s/^/exp$e /"; done; done
