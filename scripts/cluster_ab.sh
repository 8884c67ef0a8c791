#!/bin/bash
# k_tail completion: cluster barrier (libsmcsd.so) vs the per-prompt counter (libsmcsd_ab.so,
# built from the previous revision by scripts/ab_build.sh), interleaved processes.
AB=$PWD/paper_2604_15672_b200/libsmcsd_ab.so
for r in 1 2 3; do
  SMCSD_LIB_OVERRIDE=$AB python scripts/graph_ab.py | sed 's/^/counter /'
  python scripts/graph_ab.py | sed 's/^/cluster /'
done
for r in 1 2; do
  SMCSD_LIB_OVERRIDE=$AB WHICH=cfg4 python scripts/time_k1.py | sed 's/^/counter /'
  WHICH=cfg4 python scripts/time_k1.py | sed 's/^/cluster /'
done
