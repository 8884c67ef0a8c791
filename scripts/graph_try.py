#!/usr/bin/env python
"""Does CUDA-graph capture of the cfg2 step (K1 + tail, PDL edges) change the per-step time?
Eager back-to-back calls vs replays of a graph holding R steps over the 6-set ring."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
ring = [synth.lm_logits(1, 16, 8, 128256, device=dev, seed=10 + r) for r in range(6)]
ws, out = smc.Workspace(dev), smc.Outputs()
s = torch.cuda.Stream(dev)
R = 60


def steps(base):
    for i in range(R):
        smc.smcsd_step(*ring[i % 6], V=128256, eta=math.inf, step=base + i, out=out, fields=(),
                       workspace=ws, stream=s)


def timeit(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / R * 1e3)
    return sorted(ts)[len(ts) // 2]


with torch.cuda.stream(s):
    steps(0)
    torch.cuda.synchronize()
    eager = timeit(lambda: steps(0))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        steps(0)
    torch.cuda.synchronize()
    graph = timeit(lambda: g.replay())
    o1 = out.ancestors.clone()
print(f"cfg2 step: eager {eager:.2f} us/step, CUDA graph {graph:.2f} us/step (median of 5 x {R})")
