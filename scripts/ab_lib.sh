#!/bin/bash
# Interleaved A/B of libsmcsd.so (new) vs libsmcsd_ab.so (previous revision): graph_ab.py x3.
for r in 1 2 3; do
  python scripts/graph_ab.py
  SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so python scripts/graph_ab.py
done 2>&1
