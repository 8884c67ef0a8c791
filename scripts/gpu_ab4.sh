bash scripts/ab_lib.sh > gpurun_out/ab4.txt 2>&1
NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab4_trace.txt 2>&1
python -c "
import bench, torch, json
d = bench.measure_cfg2_verify(torch.device('cuda'), 6545.0)
print(json.dumps(d['plain']))
" > gpurun_out/ab4_cfg2.txt 2>&1
cat gpurun_out/ab4.txt gpurun_out/ab4_trace.txt gpurun_out/ab4_cfg2.txt
