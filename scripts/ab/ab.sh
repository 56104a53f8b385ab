# A/B of kernel-source variants on the same box: builds each variant in a copy
# of the repo under /tmp and runs a kbench command, three rounds in rotating
# order.
#   bash scripts/ab/ab.sh <csrc file name> "<kbench.py args>" a.cu b.cu [more.cu ...]
#   e.g. bash scripts/ab/ab.sh spmv.cu "spmv --n 2097152 --reps 20" /tmp/v0.cu /tmp/v1.cu
set -e
R=$(pwd); T=$1; ARGS=$2; shift 2
V=("$@"); n=${#V[@]}
for i in $(seq 0 $((n-1))); do
  d=/tmp/ab_$i; rm -rf $d; mkdir -p $d
  cp -r $R/paper_1508_06791_b200 $R/scripts $R/synth $R/include $R/bench.py $d/
  cp ${V[$i]} $d/paper_1508_06791_b200/csrc/$T
  (cd $d && python -m paper_1508_06791_b200.build > /dev/null)
done
for rep in 0 1 2; do
  for k in $(seq 0 $((n-1))); do
    i=$(( (k + rep) % n ))
    (cd /tmp/ab_$i && timeout 300 python scripts/kbench.py $ARGS 2>&1 | tail -1 | sed "s/^/$(basename ${V[$i]} .cu) /")
  done
done
