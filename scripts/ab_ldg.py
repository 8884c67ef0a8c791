#!/usr/bin/env python
"""K1 TMA ring (default) vs the LDG variant (SMCSD_K1_LDG=1, read per call): bit-identity of
the step outputs, then CUDA-graph replay timing at cfg2 and cfg4, interleaved."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")


def setmode(ldg):
    if ldg:
        os.environ["SMCSD_K1_LDG"] = "1"
    else:
        os.environ.pop("SMCSD_K1_LDG", None)


def graph_time(sets, ldg, reps, bonus=False):
    setmode(ldg)
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
    setmode(False)
    return a.elapsed_time(b) / (reps * len(sets)) * 1e3


# bit-identity
lp, lq, tok = synth.lm_logits(3, 16, 8, 128256, device=dev, seed=77)
outs = []
for ldg in (False, True):
    setmode(ldg)
    o = smc.smcsd_step(lp, lq, tok, V=128256, step=1, bonus=True)
    torch.cuda.synchronize()
    outs.append(o)
setmode(False)
same = all(torch.equal(getattr(outs[0], f), getattr(outs[1], f))
           for f in ("logw", "logw_pre", "logp_tok", "logq_tok", "ancestors", "bonus", "ess", "status"))
print("bit-identical outputs:", same, flush=True)
del lp, lq, tok
ring = [synth.lm_logits(1, 16, 8, 128256, device=dev, seed=10 + r) for r in range(6)]
big = [synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)]
for r in range(3):
    for ldg in (False, True):
        c2 = graph_time(ring, ldg, 20)
        c4 = graph_time(big * 3, ldg, 3)
        c4b = graph_time(big * 3, ldg, 3, bonus=True)
        print(f"{'LDG' if ldg else 'TMA'}  cfg2 {c2:7.2f} us   cfg4 {c4:8.1f} us   cfg4+bonus {c4b:8.1f} us", flush=True)
