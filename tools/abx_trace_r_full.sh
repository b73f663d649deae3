#!/bin/bash
# A/B of trace R (10^5 iterations, tiled) detect time across builds in tools/abx/
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for lib in "$@"; do
    echo -n "$rep $(basename $lib) "
    RESIHP_B200_LIB=$(realpath $lib) timeout 300 python tools/trace_r_tiled_time.py 2>&1 | tail -1
  done
done
