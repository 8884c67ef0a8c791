#!/bin/bash
# K1 exp-sum share on the FMA-pipe polynomial under sustained (power-capped) load: interleaved.
B=paper_2604_15672_b200
for v in 4 3 2; do
  SMCSD_AB_DEFS=SMCSD_K1_POLY_K=$v python $B/build.py > /dev/null 2>&1 && cp $B/libsmcsd_ab.so /tmp/lib_poly$v.so
done
for r in 1 2 3; do
  for v in 4 3 2; do
    echo -n "K1_POLY_K=$v  "; SMCSD_LIB_OVERRIDE=/tmp/lib_poly$v.so timeout -s KILL 120 python scripts/sustained_ab.py 2>&1 | tail -1
    sleep 2
  done
done
for r in 1 2 3; do
  for v in 1 0; do
    echo -n "poll=$v  "; SMCSD_POLL=$v timeout -s KILL 120 python scripts/sustained_ab.py 2>&1 | tail -1
    sleep 2
  done
done
