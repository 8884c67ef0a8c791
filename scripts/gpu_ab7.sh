bash scripts/ab_small.sh > gpurun_out/ab7.txt 2>&1
NOFLUSH=1 SMCSD_SMALL=1 python scripts/trace_tail.py > gpurun_out/ab7_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_latency_tail.py tests/test_gpu_multigpu.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab7_pytest.txt
cat gpurun_out/ab7.txt gpurun_out/ab7_trace.txt gpurun_out/ab7_pytest.txt
