#!/bin/bash
# One GPU call: bench, ncu launch list (share of the step), ncu --set full of the two kernels.
# Usage (under gpurun): bash scripts/gpu_profile.sh <tag>
set -x
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_rowstats|k_tail|k_kv_reindex" \
    -c 60 --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-secondary > $OUT/ncu_list_bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_rowstats -s 3 -c 1 \
    -o $OUT/prof_rowstats_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > $OUT/ncu_rowstats_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_kv_reindex -s 3 -c 1 \
    -o $OUT/prof_kv_$TAG -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-secondary > $OUT/ncu_kv_$TAG.log 2>&1
echo done
