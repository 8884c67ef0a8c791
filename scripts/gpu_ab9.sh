./scripts/ubench_lt.bin > gpurun_out/ab9_ubench.txt 2>&1
bash scripts/ab_lib.sh > gpurun_out/ab9.txt 2>&1
N=64 NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab9_trace64.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab9_pytest.txt
cat gpurun_out/ab9_ubench.txt gpurun_out/ab9.txt gpurun_out/ab9_trace64.txt gpurun_out/ab9_pytest.txt
