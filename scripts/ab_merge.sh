timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "tp or weights or step" 2>&1 | tail -2
WHICH=cfg2,cfg5,n64 bash scripts/ab_time.sh 2>&1 | tee gpurun_out/ab_merge_rows.txt
