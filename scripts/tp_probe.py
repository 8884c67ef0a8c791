#!/usr/bin/env python
"""cfg5 shape at G = 1: plain smcsd_step vs the fused-exchange smcsd_tp_step, eager back-to-back
and CUDA-graph replay (device time without host pacing), plus host enqueue cost per call.
SMCSD_LIB_OVERRIDE selects a library variant.  Usage: python scripts/tp_probe.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth
from paper_2604_15672_b200.dist import TPExchange

dev = torch.device("cuda")
P, N, K, V = 1, 64, 8, 128256
ring = [synth.lm_logits(P, N, K, V, device=dev, seed=30 + r) for r in range(3)]
# TP_EXPLICIT=1: host epoch per call (for libraries without the device-resident epoch)
ex = TPExchange.local_group(P, N, K, V, 1, device=dev,
                            device_epoch=os.environ.get("TP_EXPLICIT") != "1")[0]


def plain(i, out, ws, s=None):
    smc.smcsd_step(*ring[i % 3], V=V, step=i, out=out, fields=(), workspace=ws, stream=s)


def fused(i, out, ws, s=None):
    ex.step(*ring[i % 3], step=i, out=out, fields=(), workspace=ws, stream=s)


def eager(fn, reps=60):
    out, ws = smc.Outputs(), smc.Workspace(dev)
    for i in range(5):
        fn(i, out, ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    a.record()
    for i in range(reps):
        fn(i, out, ws)
    h1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3, (h1 - h0) / reps * 1e6


def graph(fn, per=10, reps=20):
    out, ws = smc.Outputs(), smc.Workspace(dev)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i, out, ws, s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(per):
                fn(i, out, ws, s)
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    st = out.status.cpu()
    return a.elapsed_time(b) / (reps * per) * 1e3, int(st.max())


lib = os.path.basename(smc.lib_path)
for rnd in range(2):
    for nm, fn in (("plain", plain), ("fused", fused)):
        e, h = eager(fn)
        gt, st = graph(fn)
        print(f"{lib:22s} {nm:6s} eager {e:7.2f} us (host {h:5.1f} us/call)  graph {gt:7.2f} us  status {st}")
