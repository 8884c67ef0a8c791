#!/bin/bash
# One GPU call: parity tests, smoke, then the profile script.  Usage: bash scripts/gpu_round.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log
bash scripts/gpu_profile.sh $TAG
