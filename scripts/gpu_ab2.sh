CFG4=1 bash scripts/ab_poll.sh > gpurun_out/ab2.txt 2>&1
NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab2_trace.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_latency_tail.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab2_pytest.txt
cat gpurun_out/ab2.txt gpurun_out/ab2_trace.txt gpurun_out/ab2_pytest.txt
