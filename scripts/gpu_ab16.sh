for r in 1 2 3; do python scripts/tp_ab.py; SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so python scripts/tp_ab.py; done > gpurun_out/ab16_tp.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -k "tp" tests/test_gpu_tp_ipc.py tests/test_gpu_multigpu.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/ab16_pytest.txt
cat gpurun_out/ab16_tp.txt gpurun_out/ab16_pytest.txt
