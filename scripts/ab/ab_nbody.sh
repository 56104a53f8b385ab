# A/B of nbody.cu variants on the same box: builds each variant in a copy of
# the repo under /tmp and runs the N-body kernel bench at shards 1/2/4/8,
# three rounds in rotating order.
#   bash scripts/ab/ab_nbody.sh a.cu b.cu [more.cu ...]
set -e
R=$(pwd)
run() {  # $1 = repo copy, $2 = label
  for sh in 1 2 4 8; do
    (cd $1 && timeout 300 python scripts/kbench.py nbody --shards $sh --reps 5 2>&1 | tail -1 | sed "s/^/$2 sh=$sh /")
  done
}
V=("$@"); n=${#V[@]}
for i in $(seq 0 $((n-1))); do
  d=/tmp/ab_$i; rm -rf $d; mkdir -p $d
  cp -r $R/paper_1508_06791_b200 $R/scripts $R/synth $R/include $R/bench.py $d/
  cp ${V[$i]} $d/paper_1508_06791_b200/csrc/nbody.cu
  (cd $d && python -m paper_1508_06791_b200.build > /dev/null)
done
for rep in 0 1 2; do
  for k in $(seq 0 $((n-1))); do
    i=$(( (k + rep) % n )); run /tmp/ab_$i $(basename ${V[$i]} .cu)
  done
done
