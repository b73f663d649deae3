#!/bin/bash
# A/B of trace R detect time across library builds in tools/abx/ (run on the GPU box)
cd "$(dirname "$0")/.."
n=${N:-10000}
for rep in 1 2; do
  for lib in "$@"; do
    echo -n "$rep $(basename $lib) "
    RESIHP_B200_LIB=$(realpath $lib) timeout 300 python tools/trace_r_time.py $n 2>&1 | tail -1
  done
done
