#!/bin/bash
# Interleaved A/B device timing: current libsmcsd.so vs libsmcsd_ab.so, 3 rounds.
for r in 1 2 3; do
  WHICH=${WHICH:-cfg2} python scripts/time_k1.py
  WHICH=${WHICH:-cfg2} SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so python scripts/time_k1.py
done
