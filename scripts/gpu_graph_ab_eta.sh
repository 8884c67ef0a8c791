#!/bin/bash
# scripts/gpu_graph_ab.sh at the default eta (N/2) and at eta = inf.  Usage: bash scripts/gpu_graph_ab_eta.sh lib1 lib2 ...
bash scripts/gpu_graph_ab.sh "$@"
ETA_INF=1 bash scripts/gpu_graph_ab.sh "$@"
