bash scripts/ab_lib.sh > gpurun_out/ab8.txt 2>&1
NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab8_trace.txt 2>&1
NOFLUSH=1 TRACE_LIB=paper_2604_15672_b200/libsmcsd_trace.so python scripts/trace_tail.py > /dev/null 2>&1
cat gpurun_out/ab8.txt gpurun_out/ab8_trace.txt
