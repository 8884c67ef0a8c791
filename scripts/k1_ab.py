#!/usr/bin/env python
"""One arm of a library A/B (SMCSD_LIB_OVERRIDE selects the variant): a hash of every output of
fixed steps (arms that must agree bit for bit print the same digest) and the device time per
step: cfg2 and N=64 under CUDA-graph replay (ring of 6 / 3 logit sets), cfg4 eager.
Usage (GPU): python scripts/k1_ab.py; SMCSD_LIB_OVERRIDE=.../libsmcsd_ab.so python scripts/k1_ab.py"""
import hashlib
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_15672_b200 as smc  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
arm = os.path.basename(smc.lib_path)


def digest():
    h = hashlib.sha256()
    for (P, N, K, V, dt, nd) in [(1, 16, 8, 128256, torch.bfloat16, False), (3, 7, 5, 20001, torch.float32, True),
                                 (2, 128, 2, 9000, torch.bfloat16, True), (4, 33, 3, 50000, torch.bfloat16, False)]:
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dt, seed=5 + N)
        g = torch.Generator().manual_seed(11 + N)
        ndr = torch.randint(0, K + 1, (P, N), dtype=torch.int32, generator=g) if nd else None
        prev = synth.random_logw(P, N, seed=3, sigma=0.7)
        for scheme in (0, 1):
            o = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, eta=math.inf, step=7, scheme=scheme,
                               n_drafted=None if ndr is None else ndr.to(dev), logw_prev=prev.to(dev))
            w = smc.smcsd_weights(lp.to(dev), lq.to(dev), tok.to(dev), V=V, logw_prev=prev.to(dev),
                                  n_drafted=None if ndr is None else ndr.to(dev))
            torch.cuda.synchronize()
            for t in (o.logw, o.logw_pre, o.logp_tok, o.logq_tok, o.lse, o.ess, o.wnorm, o.status, o.ancestors,
                      o.offspring, o.slot_src, o.resampled, o.n_ties, w.logw, w.lse, w.ess, w.wnorm, w.status,
                      w.logp_tok):
                h.update(t.cpu().numpy().tobytes())
    return h.hexdigest()[:16]


def graph_time(N, ring_n, reps=30):
    ring = [synth.lm_logits(1, N, 8, 128256, device=dev, seed=10 + r) for r in range(ring_n)]
    ws, out = smc.Workspace(dev), smc.Outputs()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(ring_n):
            smc.smcsd_step(*ring[i], V=128256, eta=math.inf, step=i, out=out, fields=(), workspace=ws, stream=s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for i in range(ring_n):
                smc.smcsd_step(*ring[i], V=128256, eta=math.inf, step=i, out=out, fields=(), workspace=ws, stream=s)
    g.replay()
    torch.cuda.synchronize()
    best = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        best.append(a.elapsed_time(b) / (reps * ring_n) * 1e3)
    best.sort()
    return best[len(best) // 2]


def cfg4_time():
    P, N, K, V = 64, 32, 8, 128256
    lp, lq, tok = synth.lm_logits(P, N, K, V, device=dev, seed=44)
    ws, out = smc.Workspace(dev), smc.Outputs()
    for i in range(3):
        smc.smcsd_step(lp, lq, tok, V=V, eta=math.inf, step=i, out=out, fields=(), workspace=ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(20):
        smc.smcsd_step(lp, lq, tok, V=V, eta=math.inf, step=i, out=out, fields=(), workspace=ws)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 20 * 1e3


print(f"{arm} digest {digest()}  cfg2 graph {graph_time(16, 6):7.2f} us  N64 graph {graph_time(64, 3):7.2f} us  "
      f"cfg4 {cfg4_time():8.1f} us", flush=True)
