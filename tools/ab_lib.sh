#!/bin/bash
# On the GPU box: interleaved A/B of the product library against another
# build of it (PHG_LIB_PATH), default bench line per workload.
#   tools/ab_lib.sh OTHER.so REPS WORKLOAD...
set -u
OTHER=$1; REPS=$2; shift 2
for w in "$@"; do
  for i in $(seq 1 "$REPS"); do
    for v in new old; do
      if [ $v = old ]; then export PHG_LIB_PATH=$PWD/$OTHER; else unset PHG_LIB_PATH; fi
      python bench.py --workload "$w" --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c '
import json, sys
d = json.loads(sys.stdin.read()); r = d["roofline"]
print(sys.argv[1], d["config"]["workload"][:3], d["value"], r["frac"], r["kernel_ms"], d["parity"]["ok"])' $v
    done
  done
done
