#!/bin/bash
# KV reindex variants (paper_2604_15672_b200/ab/kv_*.so): cfg3 70B in place / out of place, 2 interleaved rounds.
for r in 1 2; do
  for f in paper_2604_15672_b200/ab/kv_*.so; do
    SMCSD_LIB_OVERRIDE=$f python -c "
import bench, torch, json, os
d = bench.measure_cfg3(torch.device('cuda'), 6545.0)
print(os.path.basename('$f'), 'in_place', d['in_place']['ms_per_step'], d['in_place']['frac_of_measured'], 'out_of_place', d['out_of_place']['ms_per_step'], d['out_of_place']['frac_of_measured'], flush=True)
" 2>&1 | tail -1
  done
done
