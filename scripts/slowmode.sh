#!/bin/bash
# Frequency of the cfg4 slow mode per fresh process, default allocator vs expandable segments.
for r in $(seq 1 12); do
  WHICH=cfg4 python scripts/time_k1.py 2>&1 | grep "cfg4 " | sed 's/^/default   /'
  PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True WHICH=cfg4 python scripts/time_k1.py 2>&1 | grep "cfg4 " | sed 's/^/expandable /'
done
