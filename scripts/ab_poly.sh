#!/bin/bash
# A/B: K1 with one pair in four of its exp2 on the FMA-pipe polynomial (current build) vs all on
# MUFU (libsmcsd_ab.so), interleaved, plus the parity suite on the current build.
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
WHICH=cfg4,cfg2,cfg5,power bash scripts/ab_time.sh 2>&1 | tee gpurun_out/ab_poly.txt
