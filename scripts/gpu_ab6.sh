bash scripts/ab_lib.sh > gpurun_out/ab6.txt 2>&1
NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab6_trace.txt 2>&1
bash scripts/sanitize.sh > gpurun_out/sanitize_r02c.txt 2>&1
cat gpurun_out/ab6.txt gpurun_out/ab6_trace.txt gpurun_out/sanitize_r02c.txt
