#!/bin/bash
# K1 change vs the previous revision (libsmcsd_ab.so from scripts/ab_build.sh): cfg2 / N=64 graph
# replay (graph_ab.py) and cfg4 / cfg5-partial / PowerSMC K1 timings (time_k1.py), interleaved.
AB=$PWD/paper_2604_15672_b200/libsmcsd_ab.so
for r in 1 2 3; do
  SMCSD_LIB_OVERRIDE=$AB python scripts/graph_ab.py | sed 's/^/before /'
  python scripts/graph_ab.py | sed 's/^/after  /'
done
for r in 1 2; do
  SMCSD_LIB_OVERRIDE=$AB WHICH=cfg4,cfg5,power python scripts/time_k1.py | sed 's/^/before /'
  WHICH=cfg4,cfg5,power python scripts/time_k1.py | sed 's/^/after  /'
done
