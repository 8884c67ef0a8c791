#!/usr/bin/env python
"""Device time of the tail pieces in isolation (cfg2 shapes): smcsd_weights_combine runs
S2 (merge G parts per row) + S3 + S4 in one CTA per prompt; smcsd_resample runs S4-S7."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc

def t(fn, reps=200):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3

dev = torch.device("cuda")
for P, N, K, G in ((1, 16, 8, 16), (1, 16, 8, 1), (1, 64, 8, 8), (64, 32, 8, 16)):
    parts = torch.zeros((G, P, 2, N, K, 4), device=dev)
    parts[..., 0] = torch.randn(parts[..., 0].shape, device=dev)
    parts[..., 1] = 1.0 + torch.rand(parts[..., 1].shape, device=dev)
    parts[..., 2] = -float("inf"); parts[0, ..., 2] = parts[0, ..., 0] - 1
    tok = torch.zeros((P, N, K), dtype=torch.int32, device=dev)
    ws = smc.Workspace(dev)
    out = smc.smcsd_weights_combine(parts, tok, V=128256, workspace=ws)
    us_c = t(lambda: smc.smcsd_weights_combine(parts, tok, V=128256, out=out, workspace=ws))
    lw = torch.randn((P, N), device=dev)
    o2 = smc.smcsd_resample(lw)
    us_r = t(lambda: smc.smcsd_resample(lw, out=o2))
    empty = torch.empty(1, device=dev)
    us_e = t(lambda: empty.add_(0))
    print(f"P={P} N={N} K={K} G={G}: combine(S2-S4) {us_c:.2f} us   resample(S4-S7) {us_r:.2f} us   "
          f"(empty torch kernel {us_e:.2f} us)")
