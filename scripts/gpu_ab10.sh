python scripts/sweep_small.py > gpurun_out/ab10_sweep.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_tail_variants.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab10_pytest.txt
cat gpurun_out/ab10_sweep.txt gpurun_out/ab10_pytest.txt
