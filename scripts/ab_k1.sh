#!/bin/bash
# Interleaved A/B of libsmcsd.so vs libsmcsd_ab.so: cfg2 / N=64 graph replay, cfg4 eager (ft_ab.py), x3.
for r in 1 2 3; do
  echo -n "new "; timeout -s KILL 150 python scripts/k1_ab.py
  echo -n "ab  "; SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so timeout -s KILL 150 python scripts/k1_ab.py
done 2>&1
