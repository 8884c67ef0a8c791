#!/usr/bin/env python
"""Catch the cfg4 slow mode and find what it follows: time the same step (eager, 10 steps)
with (a) the original tensors, (b) cloned logits, (c) a fresh workspace, (d) both, (e) again (a).
Prints one line per process; run it in several fresh processes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
lp, lq, tok = synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)
ws = smc.Workspace(dev)


def tm(a_lp, a_lq, a_tok, w):
    out = smc.Outputs()
    plan = smc.StepPlan(a_lp, a_lq, a_tok, V=128256, out=out, fields=(), workspace=w)
    for i in range(3):
        plan.run(step=i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(10):
        plan.run(step=i)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 10 * 1e3


r = {"orig": tm(lp, lq, tok, ws)}
lp2, lq2 = lp.clone(), lq.clone()
r["clone_logits"] = tm(lp2, lq2, tok, ws)
ws2 = smc.Workspace(dev)
r["fresh_ws"] = tm(lp, lq, tok, ws2)
r["both"] = tm(lp2, lq2, tok, ws2)
del lp2, lq2
torch.cuda.empty_cache()
lp3 = torch.empty_like(lp); lp3.copy_(lp)
r["realloc_lp_only"] = tm(lp3, lq, tok, ws)
r["orig_again"] = tm(lp, lq, tok, ws)
print("  ".join(f"{k} {v:7.1f}" for k, v in r.items()), flush=True)
