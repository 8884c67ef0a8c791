#!/usr/bin/env python
"""Timeline of fused smcsd_step calls (cfg2 by default) from the %globaltimer trace build.
Usage (GPU): python paper_2604_15672_b200/build.py --trace && python scripts/trace_tail.py"""
import ctypes
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SMCSD_LIB_OVERRIDE"] = os.environ.get("TRACE_LIB") or os.path.join(ROOT, "paper_2604_15672_b200", "libsmcsd_trace.so")
import torch  # noqa: E402
import paper_2604_15672_b200 as smc  # noqa: E402
import synth  # noqa: E402

P, N, K, V = int(os.environ.get("P", 1)), int(os.environ.get("N", 16)), 8, 128256
dev = torch.device("cuda")
ring = [synth.lm_logits(P, N, K, V, device=dev, seed=100 + r) for r in range(6)]
lib = ctypes.CDLL(smc.lib_path)
if os.environ.get("SMCSD_SMALL") is not None:
    smc.smcsd_set_small_tail(os.environ["SMCSD_SMALL"] == "1")
buf = (ctypes.c_ulonglong * 4096)()
flush = torch.ones(64 << 20, dtype=torch.float32, device=dev)
TP = os.environ.get("TP")            # fused-exchange smcsd_tp_step at G = 1 instead of smcsd_step
B2B = int(os.environ.get("B2B", "0"))  # > 0: that many steps back to back before the traced one
if TP:
    from paper_2604_15672_b200.dist import TPExchange
    ex = TPExchange.local_group(P, N, K, V, 1, device=dev)[0]


POWER = os.environ.get("POWER")      # alpha: smcsd_powersmc_weights on [P][N][1][V] instead
if POWER:
    ring = [synth.lm_logits(P, N, 1, V, device=dev, seed=100 + r, bonus=False) for r in range(2)]


def call(it, lp, lq, tok):
    if POWER:
        return smc.smcsd_powersmc_weights(lp, V=V, alpha=float(POWER))
    if TP:
        return ex.step(lp, lq, tok, eta=math.inf, step=it, fields=())
    return smc.smcsd_step(lp, lq, tok, V=V, eta=math.inf, step=it, fields=())


for it in range(12):
    lp, lq, tok = ring[0 if os.environ.get("NOFLUSH") else it % len(ring)]
    if not os.environ.get("NOFLUSH"):
        flush_sum = flush.sum()  # read-only L2 flush (no dirty lines)
    torch.cuda.synchronize()
    lib.smcsd_trace_read(buf, 4096)
    for b in range(B2B):
        call(100 + b, *ring[b % len(ring)])
    out = call(it, lp, lq, tok)
    torch.cuda.synchronize()
lib.smcsd_trace_read(buf, 4096)
t = list(buf)
starts = [x for x in t[:1024] if x]
ends = [x for x in t[1024:2048] if x]
t0 = min(starts)
us = lambda x: (x - t0) / 1e3
s = sorted(us(x) for x in starts)
e = sorted(us(x) for x in ends)
print(f"K1 CTAs {len(starts)}: start spread {s[-1]:.2f} us; done min {e[0]:.2f} median {e[len(e)//2]:.2f} "
      f"p90 {e[int(len(e)*0.9)]:.2f} max {e[-1]:.2f} us")
names = {2060: "TP: last K1 CTA counted", 2061: "TP: system fence done", 2048: "tail CTA resident", 2049: "tail after pdl_wait", 2053: "chunk 0 S2+terms done",
         2054: "finisher rows merged", 2055: "finisher S3 done", 2050: "last CTA of prompt 0", 2051: "after S3",
         2052: "after S4-S7", 2400: "LT CTA resident", 2401: "LT inputs+warm-up", 2402: "LT S2+S3 done",
         2403: "LT S4-S7 done"}
for k, nm in names.items():
    if not t[k]:
        continue
    print(f"{nm:22s} {us(t[k]):8.2f} us")
ck = t[2200:2207]
if ck[0]:
    print("chunk 0 clocks after pdl_wait: " + "  ".join(
        f"{nm} {ck[i] - ck[0]}" for i, nm in enumerate(["wait", "flags", "S2 merge", "ell", "terms", "fence", "counter"]) if ck[i]))

fc = t[2210:2216]
if fc[0] and fc[5]:
    print("finisher clocks from rows merged: " + "  ".join(
        f"{nm} {fc[i] - fc[0]}" for i, nm in enumerate(["merged", "phase1 wait", "ell+terms", "S3+push", "arrive+stores", "barrier"]) if fc[i]))

ph = t[2300:2309]
PHASES = (["start", "exp", "prefix+ess", "anc+ties", "offspring+plan", "S7 stores", "ess/lse/wnorm"] if t[2400] else
          ["start", "M", "exp", "prefix+ess", "wnorm", "C", "u+search", "plan", "S7"])
if ph[0] and ph[1]:
    print("S4-S7 phase clocks (prompt 0, from start): " + "  ".join(
        f"{nm} {ph[i] - ph[0]}" for i, nm in enumerate(PHASES) if ph[i]))

lp_ = [t[2410 + i] for i in range(64) if t[2410 + i]]
if lp_:
    print("LT pass ends (us): " + " ".join(f"{us(x):.2f}" for x in lp_))

c = t[2490:2495]
if c[0]:
    print("LT last row clocks: poll %d  merge+ell %d | tid0: barrier->S3 done %d" % (c[1] - c[0], c[2] - c[1], c[4] - c[3]))
