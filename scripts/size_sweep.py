#!/usr/bin/env python
"""smcsd_step (S1-S7) device time vs bytes at one prompt, K=8, V=128256 bf16, N = 4 .. 256
(CUDA-graph replay of 10 steps over a ring of inputs larger than L2), and a least-squares fit
t = t0 + bytes / BW: t0 is the fixed latency (launch ramp, drain, tail), BW the streaming rate.
Usage (GPU): python scripts/size_sweep.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
V, K = 128256, 8
rows = []
for N in (4, 8, 16, 32, 64, 128, 256):
    per = 2 * N * K * V * 2
    ring_n = max(2, int(np.ceil(300e6 / per)))
    ring = [synth.lm_logits(1, N, K, V, device=dev, seed=40 + r) for r in range(ring_n)]
    ws, out = smc.Workspace(dev), smc.Outputs()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            smc.smcsd_step(*ring[i % ring_n], V=V, step=i, out=out, fields=(), workspace=ws, stream=s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(10):
                smc.smcsd_step(*ring[i % ring_n], V=V, step=i, out=out, fields=(), workspace=ws, stream=s)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 200 * 1e3
    rows.append((N, per, us))
    print(f"N={N:4d}  {per / 1e6:8.1f} MB  {us:8.2f} us  {per / us / 1e3:7.1f} GB/s", flush=True)
    del ring, g
    torch.cuda.empty_cache()
x = np.array([r[1] for r in rows], float)
y = np.array([r[2] for r in rows], float)
A = np.vstack([np.ones_like(x), x]).T
(t0, slope), *_ = np.linalg.lstsq(A, y, rcond=None)
print(f"fit: t = {t0:.2f} us + bytes / {1e-3 / slope:.0f} GB/s")
