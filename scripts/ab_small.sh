#!/bin/bash
# Interleaved A/B of the small (K1-resident) polling tail (smcsd_set_small_tail): graph_ab.py x3.
for r in 1 2 3; do
  SMCSD_SMALL=1 python scripts/graph_ab.py
  SMCSD_SMALL=0 python scripts/graph_ab.py
done 2>&1
