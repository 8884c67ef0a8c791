#!/bin/bash
WHICH=cfg4 ncu --set full --import-source on --clock-control none -k regex:k_rowstats -s 2 -c 1 \
    -o gpurun_out/prof_k1_cfg4 -f python scripts/time_k1.py > gpurun_out/prof_k1_cfg4.log 2>&1
python scripts/time_k1.py > gpurun_out/time_k1_base.txt 2>&1
