#!/bin/bash
# Interleaved cfg2 / N=64 graph-replay A/B over library variants (scripts/graph_ab.py x3 each).
# Usage: bash scripts/gpu_graph_ab.sh lib1 lib2 ...
for r in 1 2 3; do
  for l in "$@"; do SMCSD_LIB_OVERRIDE=$l python scripts/graph_ab.py; done
done 2>&1
