bash scripts/ab_lib.sh > gpurun_out/ab12.txt 2>&1
python scripts/sweep_small.py > gpurun_out/ab12_sweep.txt 2>&1
SMCSD_LIB_OVERRIDE=paper_2604_15672_b200/libsmcsd_ab.so python scripts/sweep_small.py > gpurun_out/ab12_sweep_ab.txt 2>&1
cat gpurun_out/ab12.txt gpurun_out/ab12_sweep.txt gpurun_out/ab12_sweep_ab.txt
