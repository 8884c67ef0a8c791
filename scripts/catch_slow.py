#!/usr/bin/env python
"""cfg4 K1 with the trace build: per-CTA start/end (%globaltimer) and SM id of the last call,
printed as a summary (CTAs per SM, start waves, per-CTA durations).  Run it in several fresh
processes to catch the occasional slow mode.  Usage (GPU): python scripts/catch_slow.py"""
import ctypes, os, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SMCSD_LIB_OVERRIDE"] = os.path.join(ROOT, "paper_2604_15672_b200", "libsmcsd_trace.so")
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
lp, lq, tok = synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)
ws, out = smc.Workspace(dev), smc.Outputs()
lib = ctypes.CDLL(smc.lib_path)
buf = (ctypes.c_ulonglong * 4096)()
for i in range(4):
    smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(5):
    smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
lib.smcsd_trace_read(buf, 4096)
t = list(buf)
n = 888
st, en, sm = t[:n], t[1024:1024 + n], t[3072:3072 + n]
t0 = min(st)
starts = sorted((x - t0) / 1e3 for x in st)
durs = sorted((e - s_) / 1e3 for s_, e in zip(st, en))
per_sm = collections.Counter(sm)
print(f"step {ms * 1e3:8.1f} us | CTA start: min {starts[0]:.2f} p50 {starts[n // 2]:.2f} p90 {starts[int(n * .9)]:.2f} "
      f"max {starts[-1]:.2f} us | CTA dur p10 {durs[int(n * .1)]:.1f} p50 {durs[n // 2]:.1f} max {durs[-1]:.1f} us | "
      f"SMs used {len(per_sm)}, CTAs/SM min {min(per_sm.values())} max {max(per_sm.values())}", flush=True)
