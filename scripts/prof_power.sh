#!/bin/bash
# ncu capture of the PowerSMC K1 (alpha = 4, P = 256) and the power tail; launch list too.
WHICH=power POWER_P=256 ncu --set full --import-source on --clock-control none -k regex:k_rowstats -s 2 -c 1 \
    -o gpurun_out/prof_power_k1 -f python scripts/time_k1.py > gpurun_out/prof_power_k1.log 2>&1
WHICH=power POWER_P=64 ncu --metrics gpu__time_duration.sum --clock-control none -c 24 --csv \
    --log-file gpurun_out/prof_power_launches.csv python scripts/time_k1.py > /dev/null 2>&1
