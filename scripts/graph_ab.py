#!/usr/bin/env python
"""Host cost per smcsd_step call, and cfg2 / N=64 device time per step eager vs CUDA-graph
replay (removes the host from the loop).  SMCSD_LIB_OVERRIDE selects a library variant.
Usage (GPU): python scripts/graph_ab.py"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
name = os.path.basename(smc.lib_path)
if os.environ.get("SMCSD_SMALL") is not None:                 # small (K1-resident) tail on / off
    smc.smcsd_set_small_tail(os.environ["SMCSD_SMALL"] == "1")
    name += " small=" + os.environ["SMCSD_SMALL"]
if os.environ.get("SMCSD_POLL") is not None:                  # polling tail on / off
    smc.smcsd_set_poll_tail(os.environ["SMCSD_POLL"] == "1")
    name += " poll=" + os.environ["SMCSD_POLL"]


ETA = {"eta": math.inf} if os.environ.get("ETA_INF") else {}      # default eta = N/2
if ETA:
    name += " eta=inf"


def case(label, N, ring_n=6, reps=20, P=1):
    ring = [synth.lm_logits(P, N, 8, 128256, device=dev, seed=10 + r) for r in range(ring_n)]
    ws, out = smc.Workspace(dev), smc.Outputs()
    call = lambda i: smc.smcsd_step(*ring[i % ring_n], V=128256, step=i, out=out, fields=(), workspace=ws, **ETA)
    for i in range(3):
        call(i)
    torch.cuda.synchronize()
    # host cost per call (GPU work queues up behind it)
    t = time.perf_counter()
    for i in range(200):
        call(i)
    host_us = (time.perf_counter() - t) / 200 * 1e6
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(60):
        call(i)
    b.record()
    torch.cuda.synchronize()
    eager = a.elapsed_time(b) / 60 * 1e3
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(ring_n):
            smc.smcsd_step(*ring[i], V=128256, step=i, out=out, fields=(), workspace=ws, stream=s, **ETA)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(ring_n):
                smc.smcsd_step(*ring[i], V=128256, step=i, out=out, fields=(), workspace=ws, stream=s, **ETA)
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    graph = a.elapsed_time(b) / (reps * ring_n) * 1e3
    print(f"{name:16s} {label:8s} host {host_us:6.2f} us/call  eager {eager:7.2f} us/step  graph {graph:7.2f} us/step", flush=True)


case("cfg2", 16)
case("N64", 64, ring_n=3)
if os.environ.get("CFG4"):
    case("cfg4", 32, ring_n=2, reps=5, P=64)
