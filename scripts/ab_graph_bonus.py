#!/usr/bin/env python
"""CUDA-graph replay device time of smcsd_step at cfg2 / cfg4 with and without the bonus token
(SMCSD_LIB_OVERRIDE selects a library variant)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
name = os.path.basename(smc.lib_path)


def graph_time(sets, bonus, reps):
    ws, out = smc.Workspace(dev), smc.Outputs()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i, st in enumerate(sets):
            smc.smcsd_step(*st, V=128256, step=i, out=out, fields=(), workspace=ws, stream=s, bonus=bonus)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i, st in enumerate(sets):
                smc.smcsd_step(*st, V=128256, step=i, out=out, fields=(), workspace=ws, stream=s, bonus=bonus)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (reps * len(sets)) * 1e3


ring = [synth.lm_logits(1, 16, 8, 128256, device=dev, seed=10 + r) for r in range(6)]
c2 = graph_time(ring, False, 20), graph_time(ring, True, 20)
del ring
big = [synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)]
c4 = graph_time(big * 3, False, 3), graph_time(big * 3, True, 3)
print(f"{name:16s} cfg2 {c2[0]:8.2f} us  +bonus {c2[1]:8.2f} us | cfg4 {c4[0]:9.1f} us  +bonus {c4[1]:9.1f} us", flush=True)
