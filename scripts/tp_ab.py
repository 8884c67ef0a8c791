#!/usr/bin/env python
"""Fused TP step (smcsd_tp_step, G = 1, N = 64, K = 8, V = 128256 bf16) vs the plain smcsd_step on
the same shape, both under CUDA-graph replay of a 3-set ring (median of 5 x 30 replays).
SMCSD_LIB_OVERRIDE selects a library variant.  Usage (GPU): python scripts/tp_ab.py"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth
from paper_2604_15672_b200.dist import TPExchange

dev = torch.device("cuda")
if os.environ.get("SMCSD_SMALL") is not None:                 # small (K1-resident) tails on / off
    smc.smcsd_set_small_tail(os.environ["SMCSD_SMALL"] == "1")
P, N, K, V = 1, 64, 8, 128256
ring = [synth.lm_logits(P, N, K, V, device=dev, seed=10 + r) for r in range(3)]


def graph_us(call, reps=30):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(3):
            call(i, s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(3):
                call(i, s)
    g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / (reps * 3) * 1e3)
    return sorted(out)[2]


ws, out = smc.Workspace(dev), smc.Outputs()
plain = graph_us(lambda i, s: smc.smcsd_step(*ring[i], V=V, eta=math.inf, step=i, out=out, fields=(),
                                             workspace=ws, stream=s))
ex = TPExchange.local_group(P, N, K, V, 1, device=dev)[0]
wsf, of = smc.Workspace(dev), smc.Outputs()
fused = graph_us(lambda i, s: ex.step(*ring[i], eta=math.inf, step=i, out=of, fields=(), workspace=wsf, stream=s))
ok = int(of.status.max().item()) == 0
name = os.path.basename(smc.lib_path)
print(f"{name:16s} plain {plain:7.2f} us  fused TP G=1 {fused:7.2f} us  overhead {100 * (fused / plain - 1):5.1f} %  status_ok {ok}", flush=True)
