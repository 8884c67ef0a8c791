import os, sys
sys.path.insert(0, os.getcwd())
import torch, paper_2604_15672_b200 as smc, synth
dev = torch.device("cuda")
lg, _, _ = synth.lm_logits(64, 32, 1, 128256, device=dev, seed=6, bonus=False)
ws = smc.Workspace(dev); out = smc.Outputs()
def t(fn, reps=30):
    for i in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3
for r in range(2):
    for al in (1.0, 2.0, 3.0, 4.0, 2.5, 0.5):
        us = t(lambda: smc.smcsd_powersmc_weights(lg, V=128256, alpha=al, out=out, workspace=ws))
        print(f"alpha {al}: {us:8.2f} us  {64*32*128256*2/us/1e3:7.1f} GB/s")
