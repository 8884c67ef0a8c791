#!/bin/bash
# KV reindex variants (paper_2604_15672_b200/ab/kv_*.so): the headline step (bench.py, cfg2 + 70B KV in place, N=16)
# and cfg3 (N=32), 2 interleaved rounds.
for r in 1 2; do
  for f in paper_2604_15672_b200/ab/kv_*.so; do
    v=$(SMCSD_LIB_OVERRIDE=$f python bench.py --steps 10 --warmup 3 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'])")
    c=$(SMCSD_LIB_OVERRIDE=$f python -c "
import bench, torch
d = bench.measure_cfg3(torch.device('cuda'), 6545.0)
print(d['in_place']['ms_per_step'], d['out_of_place']['ms_per_step'])
" 2>/dev/null | tail -1)
    echo "$(basename $f) headline $v cfg3(in,out) $c"
  done
done
