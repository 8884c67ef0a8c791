#!/bin/bash
# Functional check of the multi-rank bench path on ONE GPU: 2 ranks share cuda:0 over gloo
# (NCCL refuses two ranks on one device).  Timing from this run is not a bench value.
SMCSD_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 10 --warmup 3 \
    > gpurun_out/multirank.json 2> gpurun_out/multirank.err
echo "rc=$?"
