#!/usr/bin/env python
"""Latency tail (smcsd_lt.cuh) vs the two-kernel path (K1 -> k_tail), same library, toggled with
smcsd_set_latency_tail: (1) bit-identity of every output on a set of shapes, (2) CUDA-graph
replay time per step, interleaved.  Usage (GPU): python scripts/lt_ab.py [--no-timing]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2604_15672_b200 as smc  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda")
FIELDS = ("logw", "logw_pre", "logp_tok", "logq_tok", "lse", "ess", "wnorm", "status", "ancestors",
          "offspring", "slot_src", "resampled", "n_ties")


def outputs(o):
    return {f: getattr(o, f).clone() for f in FIELDS if getattr(o, f, None) is not None}


def parity():
    bad = 0
    cases = [  # P, N, K, V, dtype, extra
        (1, 16, 8, 128256, torch.bfloat16, {}),
        (1, 4, 4, 1000, torch.float32, {}),
        (3, 32, 8, 50001, torch.bfloat16, {}),
        (2, 7, 3, 20001, torch.float32, {"scheme": smc.SMCSD_MULTINOMIAL}),
        (1, 1, 1, 7, torch.float32, {}),
        (4, 32, 16, 128256, torch.bfloat16, {"eta": None}),
        (2, 12, 8, 131072, torch.bfloat16, {}),
        (3, 9, 5, 8193, torch.float32, {}),
        (5, 8, 16, 32000, torch.bfloat16, {"alpha": 0.7, "inv_temp_p": 1.3}),
    ]
    for P, N, K, V, dt, extra in cases:
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dt, seed=900 + N + V, bonus=False)
        lp, lq, tok = lp.to(dev), lq.to(dev), tok.to(dev)
        nd = torch.randint(0, K + 1, (P, N), dtype=torch.int32, device=dev)
        prev = torch.randn(P, N, device=dev) * 0.3
        for mode in ("step", "weights"):
            for ndv in (None, nd):
                kw = dict(V=V, n_drafted=ndv, logw_prev=prev, step=3, eta=extra.get("eta", math.inf))
                kw.update({k: v for k, v in extra.items() if k != "eta"})
                res = []
                for lt in (False, True, False, True):
                    smc.smcsd_set_latency_tail(lt)
                    ws = smc.Workspace(dev)
                    if mode == "step":
                        o = smc.smcsd_step(lp, lq, tok, workspace=ws, **kw)
                    else:
                        kw2 = {k: v for k, v in kw.items() if k in ("V", "n_drafted", "logw_prev", "alpha", "inv_temp_p")}
                        o = smc.smcsd_weights(lp, lq, tok, workspace=ws, **kw2)
                    torch.cuda.synchronize()
                    res.append(outputs(o))
                ok = True
                for f in res[0]:
                    for r in res[1:]:
                        a, b = res[0][f], r[f]
                        same = torch.equal(a.view(torch.uint8) if a.is_floating_point() else a,
                                           b.view(torch.uint8) if b.is_floating_point() else b)
                        if not same:
                            ok = False
                            print(f"  MISMATCH {mode} P={P} N={N} K={K} V={V} nd={ndv is not None} field {f}")
                bad += not ok
                print(f"parity {mode:7s} P={P} N={N:2d} K={K:2d} V={V:6d} {str(dt)[6:]:8s} nd={ndv is not None!s:5s} "
                      f"{'ok' if ok else 'FAIL'}", flush=True)
    smc.smcsd_set_latency_tail(False)
    return bad


def timing(label, P, N, ring_n=6, reps=20, K=8, V=128256):
    ring = [synth.lm_logits(P, N, K, V, device=dev, seed=10 + r, bonus=False) for r in range(ring_n)]
    res = {}
    for lt in (False, True, False, True, False, True):
        smc.smcsd_set_latency_tail(lt)
        ws, out = smc.Workspace(dev), smc.Outputs()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            for i in range(ring_n):
                smc.smcsd_step(*ring[i], V=V, step=i, eta=math.inf, out=out, fields=(), workspace=ws, stream=s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for i in range(ring_n):
                    smc.smcsd_step(*ring[i], V=V, step=i, eta=math.inf, out=out, fields=(), workspace=ws, stream=s)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) / (reps * ring_n) * 1e3
        res.setdefault(lt, []).append(us)
        del g
    smc.smcsd_set_latency_tail(False)
    f = lambda v: " ".join(f"{x:8.2f}" for x in v)
    print(f"{label:10s} two-kernel {f(res[False])} us   LT {f(res[True])} us", flush=True)


if __name__ == "__main__":
    nbad = parity() if "--no-parity" not in sys.argv else 0
    print(f"parity failures: {nbad}", flush=True)
    if "--no-timing" not in sys.argv:
        timing("cfg2", 1, 16)
        timing("N32", 1, 32)
        timing("N4K16", 1, 4, K=16)
        timing("P8N16", 8, 16, ring_n=3)
        timing("cfg4", 64, 32, ring_n=2, reps=5)
