#!/bin/bash
# time every library variant in the package dir on cfg4/cfg2/cfg5 shapes
OUT=gpurun_out/${1:-sweep}.txt
: > $OUT
for lib in paper_2604_15672_b200/libsmcsd*.so; do
  case $lib in *trace*) continue;; esac
  SMCSD_LIB_OVERRIDE=$PWD/$lib python scripts/time_k1.py >> $OUT 2>&1
done
