#!/usr/bin/env python
"""Does the cfg4 slow mode follow the workspace (work counter / partials address)?  One set of
inputs, a fresh Workspace per trial, CUDA-graph replay timing."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
lp, lq, tok = synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)
keep = []
for trial in range(int(os.environ.get("TRIALS", 10))):
    ws, out = smc.Workspace(dev), smc.Outputs()
    buf = ws.get(64, 32, 8, 128256)
    keep.append(ws)                                   # keep every workspace alive: new addresses
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        smc.smcsd_step(lp, lq, tok, V=128256, out=out, fields=(), workspace=ws, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(3):
                smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws, stream=s)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    print(f"trial {trial}: {a.elapsed_time(b) / 9 * 1e3:8.1f} us  ws@{buf.data_ptr():#x}", flush=True)
