#!/usr/bin/env python
"""SURVEY 8(d) secondary sweep: smcsd_step (S1-S7) over the paper's (N, K) operating points
 and prompt batch P in {1, 4, 8, 16}, V = 128256 bf16.
Device time per step (CUDA events, back-to-back calls over a 2-set ring), achieved GB/s of the
algorithmic logit bytes 2*N*K*V*2*P, fraction of the measured copy peak.  Context curve only."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_15672_b200 as smc
import synth

def _measured_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else the profiling guide's fallback."""
    import json
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


PEAK = _measured_peak()
try:
    PEAK = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
NK = [(12, 8), (8, 16), (6, 12), (12, 16), (4, 32), (8, 32), (4, 64), (16, 12), (8, 48), (8, 8),
      (4, 16), (8, 26)]
V = 128256
dev = torch.device("cuda")
print(f"{'N':>3} {'K':>3} {'P':>3} {'us/step':>9} {'GB/s':>8} {'frac':>6}")
for P in (1, 4, 8, 16):
    for N, K in NK:
        ring = [synth.lm_logits(P, N, K, V, device=dev, seed=31 + r) for r in range(2)]
        ws, out = smc.Workspace(dev), smc.Outputs()
        fn = lambda i: smc.smcsd_step(*ring[i % 2], V=V, eta=math.inf, step=i, out=out, fields=(),
                                      workspace=ws)
        for i in range(4):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 40
        a.record()
        for i in range(reps):
            fn(i)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / reps * 1e3
        gbs = 2 * N * K * V * 2 * P / (us * 1e-6) / 1e9
        print(f"{N:>3} {K:>3} {P:>3} {us:9.2f} {gbs:8.1f} {gbs / PEAK:6.3f}", flush=True)
        del ring
        torch.cuda.empty_cache()
