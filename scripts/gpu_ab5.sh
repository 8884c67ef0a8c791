bash scripts/ab_lib.sh > gpurun_out/ab5.txt 2>&1
NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab5_trace.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab5_pytest.txt
cat gpurun_out/ab5.txt gpurun_out/ab5_trace.txt gpurun_out/ab5_pytest.txt
