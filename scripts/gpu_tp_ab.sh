#!/bin/bash
# Interleaved fused-TP A/B over library variants (scripts/tp_ab.py x3 each).  Usage: bash scripts/gpu_tp_ab.sh lib1 lib2 ...
for r in 1 2 3; do
  for l in "$@"; do SMCSD_LIB_OVERRIDE=$l python scripts/tp_ab.py; done
done 2>&1
