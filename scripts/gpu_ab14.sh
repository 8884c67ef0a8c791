timeout 900 python -m pytest tests/test_gpu_parity.py -k "tp" -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab14_pytest_tp.txt
timeout 900 python -m pytest tests/test_gpu_tp_ipc.py tests/test_gpu_multigpu.py -m gpu -x -q 2>&1 | tail -2 >> gpurun_out/ab14_pytest_tp.txt
for r in 1 2; do python scripts/tp_ab.py; SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so python scripts/tp_ab.py; done > gpurun_out/ab14_tp.txt 2>&1
TP=1 N=64 NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/ab14_trace_tp.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab14_pytest.txt
cat gpurun_out/ab14_pytest_tp.txt gpurun_out/ab14_tp.txt gpurun_out/ab14_trace_tp.txt gpurun_out/ab14_pytest.txt
