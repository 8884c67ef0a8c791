#!/usr/bin/env python
"""Sustained cfg4 smcsd_step (CUDA-graph replay) for ~DURATION s: per-second step time next to
GPU / HBM temperature, SM and memory clocks and clock-event reasons (NVML)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2604_15672_b200 as smc
import synth

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


def temps():
    gpu = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
    try:
        fv = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_MEMORY_TEMP])[0]
        mem = fv.value.uiVal if fv.nvmlReturn == 0 else -1
    except Exception:
        mem = -1
    return gpu, mem


dev = torch.device("cuda")
lp, lq, tok = synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)
ws, out = smc.Workspace(dev), smc.Outputs()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    smc.smcsd_step(lp, lq, tok, V=128256, out=out, fields=(), workspace=ws, stream=s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(10):
            smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws, stream=s)
t_end = time.time() + float(os.environ.get("DURATION", 40))
print("sec  us/step  gpuC memC  watts  sm_mhz mem_mhz reasons", flush=True)
t0 = time.time()
while time.time() < t_end:
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    n = 0
    ts = time.time()
    while time.time() - ts < 1.0:
        g.replay()
        n += 10
        if n % 200 == 0:
            torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1e3
    gt, mt = temps()
    print(f"{time.time() - t0:4.0f} {us:8.1f}  {gt:4d} {mt:4d}  {pynvml.nvmlDeviceGetPowerUsage(h) / 1000:5.0f}  {pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM):6d} "
          f"{pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM):6d} {hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))}", flush=True)
