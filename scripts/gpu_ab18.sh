bash scripts/kv_ab.sh > gpurun_out/kv_ab2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -k "kv or reindex" tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -2 > gpurun_out/kv_ab2_pytest.txt
cat gpurun_out/kv_ab2.txt gpurun_out/kv_ab2_pytest.txt
