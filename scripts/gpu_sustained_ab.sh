#!/bin/bash
# cfg4 burst and sustained (power-capped) timing over library variants, interleaved (scripts/sustained_ab.py).
# Usage: bash scripts/gpu_sustained_ab.sh lib1 lib2 ...
for r in $(seq 1 ${REPS:-3}); do
  for l in "$@"; do
    echo -n "$(basename $l)  "; SMCSD_LIB_OVERRIDE=$l timeout -s KILL 120 python scripts/sustained_ab.py 2>&1 | tail -1
    sleep 2
  done
done
