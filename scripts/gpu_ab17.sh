bash scripts/ab_lib.sh > gpurun_out/ab17.txt 2>&1
for i in 1 2; do NOFLUSH=1 python scripts/trace_tail.py; done > gpurun_out/ab17_trace.txt 2>&1
python scripts/sweep_small.py > gpurun_out/ab17_sweep.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_tail_variants.py tests/test_gpu_parity.py tests/test_gpu_multigpu.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab17_pytest.txt
cat gpurun_out/ab17.txt gpurun_out/ab17_trace.txt gpurun_out/ab17_sweep.txt gpurun_out/ab17_pytest.txt
