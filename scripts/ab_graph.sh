#!/bin/bash
for r in 1 2 3; do
  python scripts/graph_ab.py
  SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so python scripts/graph_ab.py
done 2>&1 | tee gpurun_out/ab_graph.txt
