#!/usr/bin/env python
"""Does the cfg4 step time depend on where the 8.9 GB of logits land?  Re-allocate the inputs
several times in one process (releasing memory to the driver in between) and time each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
ws, out = smc.Workspace(dev), smc.Outputs()
base = synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)
for trial in range(int(os.environ.get("TRIALS", 8))):
    lp, lq, tok = (t.clone() for t in base) if trial else base
    fn = lambda i: smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws)
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(10):
        fn(i)
    b.record()
    torch.cuda.synchronize()
    print(f"trial {trial}: {a.elapsed_time(b) / 10 * 1e3:8.1f} us  lp@{lp.data_ptr():#x}", flush=True)
    if trial:
        del lp, lq, tok
    torch.cuda.empty_cache()
