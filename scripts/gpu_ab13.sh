bash scripts/ab_lib.sh > gpurun_out/ab13.txt 2>&1
python scripts/sweep_small.py > gpurun_out/ab13_sweep.txt 2>&1
N=64 NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab13_trace64.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_tail_variants.py tests/test_gpu_parity.py tests/test_gpu_multigpu.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab13_pytest.txt
cat gpurun_out/ab13.txt gpurun_out/ab13_sweep.txt gpurun_out/ab13_trace64.txt gpurun_out/ab13_pytest.txt
