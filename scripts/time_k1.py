#!/usr/bin/env python
"""Device time of smcsd_step / smcsd_weights_partial on cfg4 / cfg2 / cfg5 shapes (events over
back-to-back calls).  SMCSD_LIB_OVERRIDE selects a library variant.  Usage: python scripts/time_k1.py"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth

dev = torch.device("cuda")
which = os.environ.get("WHICH", "cfg4,cfg2,cfg5,power").split(",")

try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    def _clk():
        return (pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_MEM),
                hex(pynvml.nvmlDeviceGetCurrentClocksEventReasons(_h)))
except Exception:
    _clk = lambda: None


def t(fn, reps, warm=3):
    for i in range(warm): fn(i)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(reps): fn(i)
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def _measured_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written), else the profiling guide's fallback."""
    import json
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


PEAK = _measured_peak()
res = {}
if "cfg4" in which:
    lp, lq, tok = synth.lm_logits(64, 32, 8, 128256, device=dev, seed=4)
    ws = smc.Workspace(dev); out = smc.Outputs()
    ms = t(lambda i: smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws), 10)
    res["cfg4"] = (ms, 8405475328 / ms / 1e6)
    ms = t(lambda i: smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws, bonus=True), 10)
    res["cfg4+bonus"] = (ms, (8405475328 + 2048 * 128256 * 2) / ms / 1e6)
    del lp, lq, tok; torch.cuda.empty_cache()
if "cfg2" in which:
    ring = [synth.lm_logits(1, 16, 8, 128256, device=dev, seed=10 + r) for r in range(6)]
    ws = smc.Workspace(dev); out = smc.Outputs()
    ms = t(lambda i: smc.smcsd_step(*ring[i % 6], V=128256, step=i, out=out, fields=(), workspace=ws), 60)
    res["cfg2"] = (ms, 65667776 / ms / 1e6)
    ms = t(lambda i: smc.smcsd_step(*ring[i % 6], V=128256, step=i, out=out, fields=(), workspace=ws, bonus=True), 60)
    res["cfg2+bonus"] = (ms, (65667776 + 16 * 128256 * 2) / ms / 1e6)
    del ring; torch.cuda.empty_cache()
if "cfg5" in which:
    lp, lq, tok = synth.lm_logits(1, 64, 8, 128256, device=dev, seed=5)
    ws = smc.Workspace(dev)
    part = torch.empty((1, 2, 64, 8, 4), device=dev)
    ms = t(lambda i: smc.smcsd_weights_partial(lp, lq, tok, v_begin=0, v_len=128256, partials=part, workspace=ws), 30)
    res["cfg5-partial-G1"] = (ms, 262668288 / ms / 1e6)
if "n64" in which:
    ring = [synth.lm_logits(1, 64, 8, 128256, device=dev, seed=20 + r) for r in range(3)]
    ws = smc.Workspace(dev); out = smc.Outputs()
    ms = t(lambda i: smc.smcsd_step(*ring[i % 3], V=128256, step=i, out=out, fields=(), workspace=ws), 30)
    res["N64-step"] = (ms, 262668288 / ms / 1e6)
    del ring; torch.cuda.empty_cache()
if "fp32" in which:
    # cfg2 / cfg4 shapes with fp32 logits (2x the bytes of bf16)
    for nm, P_ in (("fp32-cfg2", 1), ("fp32-cfg4", 16)):
        lp, lq, tok = synth.lm_logits(P_, 32 if P_ > 1 else 16, 8, 128256, dtype=torch.float32, device=dev, seed=8)
        ws = smc.Workspace(dev); out = smc.Outputs()
        ms = t(lambda i: smc.smcsd_step(lp, lq, tok, V=128256, step=i, out=out, fields=(), workspace=ws), 10)
        byts = 2 * lp.shape[0] * lp.shape[1] * 8 * 128256 * 4
        res[nm] = (ms, byts / ms / 1e6)
        del lp, lq, tok; torch.cuda.empty_cache()
if "tp" in which:
    # S10 fused exchange at G = 1 (smcsd_tp_step: K1 pushes partials, tail waits on the flag)
    from paper_2604_15672_b200.dist import TPExchange
    lp, lq, tok = synth.lm_logits(1, 64, 8, 128256, device=dev, seed=5)
    ex = TPExchange.local_group(1, 64, 8, 128256, 1, device=dev)[0]
    ws = smc.Workspace(dev); out = smc.Outputs()
    ms = t(lambda i: ex.step(lp, lq, tok, step=i, out=out, fields=(), workspace=ws), 30)
    res["tp-fused-G1"] = (ms, 262668288 / ms / 1e6)
    del lp, lq, tok; torch.cuda.empty_cache()
if "power" in which:
    PP = int(os.environ.get("POWER_P", "64"))
    lg, _, _ = synth.lm_logits(PP, 32, 1, 128256, device=dev, seed=6, bonus=False)
    ws = smc.Workspace(dev); out = smc.Outputs()
    for al in (4.0, 2.5):
        ms = t(lambda i: smc.smcsd_powersmc_weights(lg, V=128256, alpha=al, out=out, workspace=ws), 30)
        res[f"power-P{PP}-a{al}"] = (ms, PP * 32 * 128256 * 2 / ms / 1e6)
    del lg; torch.cuda.empty_cache()
for k, (ms, gbs) in res.items():
    print(f"{os.path.basename(smc.lib_path):24s} {k:16s} {ms * 1e3:9.2f} us  {gbs:8.1f} GB/s  ({gbs / PEAK:.3f} of measured)  clk {_clk()}")
