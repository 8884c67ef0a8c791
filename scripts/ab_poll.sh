#!/bin/bash
# Interleaved A/B of the polling tail (smcsd_set_poll_tail) in one library: graph_ab.py x3.
for r in 1 2 3; do
  SMCSD_POLL=1 python scripts/graph_ab.py
  SMCSD_POLL=0 python scripts/graph_ab.py
done 2>&1
