#!/bin/bash
# Launch list (per-kernel durations) of the mid-size paths: cfg5 partial, PowerSMC, cfg2.
WHICH=cfg5,power,cfg2 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,dram__bytes_read.sum \
    --clock-control none -k regex:"k_rowstats|k_tail|k_merge|k_power" -c 400 --csv \
    --log-file gpurun_out/mid_launches.csv python scripts/time_k1.py > gpurun_out/mid_time.log 2>&1
WHICH=cfg5,power,cfg2 python scripts/time_k1.py >> gpurun_out/mid_time.log 2>&1
