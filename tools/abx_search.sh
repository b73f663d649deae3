#!/bin/bash
# A/B of the re-plan search eval across library builds in tools/abx/ (run on the GPU box)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for lib in "$@"; do
    echo -n "$rep $(basename $lib) "
    RESIHP_B200_LIB=$(realpath $lib) timeout 600 python tools/search_eval_time.py 2>&1 | tail -1
  done
done
