#!/usr/bin/env python
"""PowerSMC weights (64 prompts x N=32, V=128256 bf16) for a few alpha, one library variant
(SMCSD_LIB_OVERRIDE).  Usage (GPU): python scripts/pw_ab.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
lg, _, _ = synth.lm_logits(64, 32, 1, 128256, device=dev, seed=6, bonus=False)
ws, out = smc.Workspace(dev), smc.Outputs()
peak = 6541.8


def t(fn, reps=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


name = os.path.basename(smc.lib_path)
for al in (2.7, 1.3, 4.0):
    us = t(lambda: smc.smcsd_powersmc_weights(lg, V=128256, alpha=al, out=out, workspace=ws))
    gbs = 64 * 32 * 128256 * 2 / us / 1e3
    print(f"{name:28s} alpha {al}: {us:8.2f} us  {gbs:7.1f} GB/s  {gbs / peak:.3f}", flush=True)
