#!/usr/bin/env python
"""cfg4 (64 prompts x N=32 x K=8, V=128256 bf16) under sustained load: ~SETTLE s of back-to-back
steps (the board reaches its power cap), then ~1 s timed, SM clock / power / reasons sampled.
SMCSD_LIB_OVERRIDE selects a library variant.  Usage (GPU): python scripts/sustained_ab.py"""
import math, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2604_15672_b200 as smc
import synth

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
dev = torch.device("cuda")
if os.environ.get("SMCSD_POLL") is not None:                  # polling tail on / off
    smc.smcsd_set_poll_tail(os.environ["SMCSD_POLL"] == "1")
P, N, K, V = 64, 32, 8, 128256
lp, lq, tok = synth.lm_logits(P, N, K, V, device=dev, seed=4)
ws, out = smc.Workspace(dev), smc.Outputs()
fn = lambda i: smc.smcsd_step(lp, lq, tok, V=V, eta=math.inf, step=i, out=out, fields=(), workspace=ws)
for i in range(3):
    fn(i)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(10):
    fn(i)
b.record()
torch.cuda.synchronize()
burst = a.elapsed_time(b) / 10 * 1e3
t_end = time.time() + float(os.environ.get("SETTLE", 3.0))
i = 0
while time.time() < t_end:
    fn(i); i += 1
    if i % 50 == 0:
        torch.cuda.synchronize()
clk, pw = [], []
a.record()
n = 700
for k in range(n):
    fn(k)
    if k % 100 == 0:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
b.record()
torch.cuda.synchronize()
sus = a.elapsed_time(b) / n * 1e3
byts = P * 2 * N * K * V * 2
name = os.path.basename(smc.lib_path) + (" poll=" + os.environ["SMCSD_POLL"] if os.environ.get("SMCSD_POLL") else "")
print(f"{name:40s} burst {burst:7.1f} us ({byts / burst / 1e3 / 6451.5:.3f})  sustained {sus:7.1f} us "
      f"({byts / sus / 1e3 / 6451.5:.3f})  sm {statistics.median(clk):.0f} MHz  {statistics.median(pw):.0f} W", flush=True)
