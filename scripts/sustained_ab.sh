#!/bin/bash
# K1 ring shapes under sustained (power-capped) load: CTAs/SM x stages variants, interleaved.
B=paper_2604_15672_b200
for v in "SMCSD_K1_MINB=6,SMCSD_K1_STAGES=2" "SMCSD_K1_MINB=4,SMCSD_K1_STAGES=3" "SMCSD_K1_MINB=5,SMCSD_K1_STAGES=2" "SMCSD_K1_MINB=3,SMCSD_K1_STAGES=4"; do
  SMCSD_AB_DEFS=$v python $B/build.py > /dev/null 2>&1 && cp $B/libsmcsd_ab.so /tmp/lib_$(echo $v | tr ',=' '__').so
done
for r in 1 2; do
  for v in "SMCSD_K1_MINB=6,SMCSD_K1_STAGES=2" "SMCSD_K1_MINB=4,SMCSD_K1_STAGES=3" "SMCSD_K1_MINB=5,SMCSD_K1_STAGES=2" "SMCSD_K1_MINB=3,SMCSD_K1_STAGES=4"; do
    echo -n "$v  "; SMCSD_LIB_OVERRIDE=/tmp/lib_$(echo $v | tr ',=' '__').so timeout -s KILL 120 python scripts/sustained_ab.py 2>&1 | tail -1
    sleep 2
  done
done
