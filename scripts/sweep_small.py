#!/usr/bin/env python
"""The paper's batch-1 operating points (N, K), V=128256 bf16: CUDA-graph time
per smcsd_step with the small (K1-resident) polling tail on / off, interleaved in one process.
Usage (GPU): python scripts/sweep_small.py"""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
V = 128256
POINTS = [(12, 8), (8, 16), (6, 12), (12, 16), (4, 32), (8, 32), (4, 64), (16, 12), (8, 48), (8, 8), (4, 16), (8, 26)]


def graph_us(N, K, ring, R=24, reps=5):
    ws, out = smc.Workspace(dev), smc.Outputs()
    gs = torch.cuda.Stream()
    gs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        for i in range(len(ring)):
            smc.smcsd_step(*ring[i], V=V, eta=math.inf, step=i, out=out, fields=(), workspace=ws, stream=gs)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=gs):
            for i in range(R):
                smc.smcsd_step(*ring[i % len(ring)], V=V, eta=math.inf, step=i, out=out, fields=(), workspace=ws, stream=gs)
    g.replay()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); g.replay(); b.record(); torch.cuda.synchronize()
        t.append(a.elapsed_time(b) / R * 1e3)
    del g
    return statistics.median(t)


for N, K in POINTS:
    ring = [synth.lm_logits(1, N, K, V, device=dev, seed=300 + r, bonus=False) for r in range(3)]
    res = {True: [], False: []}
    for on in (True, False, True, False):
        smc.smcsd_set_small_tail(on)
        res[on].append(graph_us(N, K, ring))
    smc.smcsd_set_small_tail(True)
    print(f"N={N:2d} K={K:2d}  small {min(res[True]):7.2f} us   256-thread polling {min(res[False]):7.2f} us", flush=True)
    del ring
