#!/usr/bin/env python
"""Where the host time of one smcsd_step call goes (GPU box): full binding call, the bare
ctypes call with prepared arguments, and the pieces (stream lookup, data_ptr)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
lp, lq, tok = synth.lm_logits(1, 16, 8, 128256, device=dev, seed=1)
ws, out = smc.Workspace(dev), smc.Outputs()
smc.smcsd_step(lp, lq, tok, V=128256, out=out, fields=(), workspace=ws)
torch.cuda.synchronize()


def t(label, fn, n=2000):
    for _ in range(50):
        fn()
    a = time.perf_counter()
    for _ in range(n):
        fn()
    us = (time.perf_counter() - a) / n * 1e6
    torch.cuda.synchronize()
    print(f"{label:40s} {us:8.2f} us")


t("smcsd_step (binding)", lambda: smc.smcsd_step(lp, lq, tok, V=128256, out=out, fields=(), workspace=ws), 500)
t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream)
t("tensor.data_ptr()", lambda: lp.data_ptr())
t("ws.get", lambda: ws.get(1, 16, 8, 128256))
if hasattr(smc, "StepPlan"):
    plan = smc.StepPlan(lp, lq, tok, V=128256, out=out, fields=(), workspace=ws)
    t("StepPlan.run", lambda: plan.run(step=3), 500)
    t("StepPlan.run(inputs)", lambda: plan.run(lp, lq, tok, step=3), 500)
