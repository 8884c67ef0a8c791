# latency-tail A/B (scripts/lt_ab.py), traces, warp_tail microbenchmark, GPU tests
set -x
./scripts/ubench_lt.bin > gpurun_out/lt_ubench.txt 2>&1
timeout 300 python scripts/lt_ab.py > gpurun_out/lt_ab.txt 2>&1
SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so timeout 300 python scripts/lt_ab.py --no-parity > gpurun_out/lt_ab_dry.txt 2>&1
NOFLUSH=1 SMCSD_LT=1 python scripts/trace_tail.py > gpurun_out/lt_trace_noflush.txt 2>&1
NOFLUSH=1 python scripts/trace_tail.py > gpurun_out/lt_trace_noflush_off.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/lt_pytest.txt 2>&1
cat gpurun_out/lt_ubench.txt; grep -v "^parity step\|^parity weights" gpurun_out/lt_ab.txt; cat gpurun_out/lt_ab_dry.txt gpurun_out/lt_trace_noflush.txt gpurun_out/lt_trace_noflush_off.txt; tail -3 gpurun_out/lt_pytest.txt
