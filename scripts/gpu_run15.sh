set -x
for v in "4 1" "4 10" "4 8" "3 1" "3 12" "5 1" "2 1"; do set -- $v; JACC_NBODY_PAIRS=$1 JACC_NBODY_MINB=$2 timeout 120 python scripts/kbench.py nbody --reps 4 | sed "s/^/P=$1 MB=$2 /"; done
