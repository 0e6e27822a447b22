#!/bin/bash
# A/B of device solve time: tools/ab_solve.sh <config> <solves> <libA> <libB> ... (alternating, twice)
cfg=$1; n=$2; shift 2
for rep in 1 2; do
  for lib in "$@"; do
    echo "== $lib"
    LR_LIB=$lib python tools/prof_solve.py --config $cfg --solves $n 2>&1 | grep device_ms
  done
done
