#!/bin/bash
# A/B of a K2-tail change: GPU tests on the current build, interleaved timing vs libsmcsd_ab.so,
# %globaltimer traces of the current build (cfg2, N=64).
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
WHICH=cfg2,n64,cfg5,cfg4 bash scripts/ab_time.sh 2>&1 | tee gpurun_out/ab_tail.txt
timeout 120 python scripts/trace_tail.py 2>&1 | tee gpurun_out/trace_tail.txt
N=64 timeout 120 python scripts/trace_tail.py 2>&1 | sed 's/^/N64: /' | tee -a gpurun_out/trace_tail.txt
