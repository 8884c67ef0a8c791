bash scripts/ab_lib.sh > gpurun_out/ab11.txt 2>&1
NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab11_trace.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab11_pytest.txt
cat gpurun_out/ab11.txt gpurun_out/ab11_trace.txt gpurun_out/ab11_pytest.txt
