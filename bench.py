#!/usr/bin/env python
"""bench.py -- SMC-SD verify + resample hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--no-secondary] [--no-cpu-baseline]

A step is one pass of the whole hot path over one batch of
synthetic input.  Default workload (configs[1] of BASELINE.json, one prompt per GPU):
  verify + resample  V=128256, N=16, K=8, bf16 logits   (smcsd_step: S1-S7, K1 + K2)
  + KV reindex of Llama-3.1-70B-shaped per-particle KV caches (80 L x 2 x 8 KV heads x
    seq 2048 x d 128 bf16 = 640 MiB per particle) with the in-place slot plan (S8)
  + token-history reindex (S9).
eta = +inf forces a resample every step (worst case).  Logits come from a ring of 6 input
sets (394 MB > 126 MB L2); the KV caches (10.7 GB) exceed L2.  Timing: W untimed steps, then K
steps bracketed by barrier + synchronize, CUDA events on the launching stream, max over ranks.
For N > 1 (torchrun) each rank runs its own prompt (global prompt index = rank): weak scaling,
no data-path collective.  The line's `secondary` object adds cfg4 (64 prompts), cfg5 (vocab-
sharded TP: the fused peer-memory exchange, with the NCCL all-gather / all-reduce forms as
baselines), cfg3 (70B KV reindex, dense and paged), the cfg2 verify path alone and PowerSMC.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SMC verify+resample steps/s; achieved HBM GB/s vs B200 peak"
NORTH_STAR_TBS = 8.0
KV70B = dict(L=80, H=8, S=2048, d=128)
COLD_READ_FLOOR_US = 12.70    # cold 64 MB read, no compute, best config (profiles/r01_ubench_stream.txt)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def traffic_table():
    """dram bytes per launch per kernel from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and clocks-event reasons with NVML while the timed region runs."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
             0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
             0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            h = None
            try:
                uuid = str(torch.cuda.get_device_properties(device_index).uuid)
                h = pynvml.nvmlDeviceGetHandleByUUID(("GPU-" + uuid) if not uuid.startswith("GPU") else uuid)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.h, self.nv = h, pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        names = [n for b, n in self.NAMES.items() if self.reasons & b and b != 0x1]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


# ------------------------------------------------------------------------------ env
def dist_env(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = os.environ.get("SMCSD_BENCH_BACKEND", "nccl")   # gloo: functional test only
        if args.impl == "reference" or backend == "gloo":
            if args.impl != "reference":
                if torch.cuda.device_count() == 0:
                    raise SystemExit("bench.py: our arm runs the CUDA path and this box has no GPU "
                                     "(--impl reference runs the CPU oracle arm)")
                torch.cuda.set_device(local % torch.cuda.device_count())
            dist.init_process_group("gloo")
        else:
            if torch.cuda.device_count() < world:
                raise SystemExit(f"bench.py: {world} NCCL ranks need {world} GPUs, this box has "
                                 f"{torch.cuda.device_count()} (SMCSD_BENCH_BACKEND=gloo shares one)")
            # NCCL's INIT log (communicator size, NVLink / NVLS transport) on stderr, so the one
            # JSON line on stdout stays clean
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ------------------------------------------------------------------------------ workloads
class Cfg2Step:
    """configs[1]: verify+resample (N=16, K=8, V=128256 bf16) + 70B-KV in-place reindex."""
    name = "cfg2"

    def __init__(self, dev, rank, args, N=16, K=8, V=128256, P=1, ring=6, kv=True):
        import torch
        import paper_2604_15672_b200 as smc
        import synth
        self.smc, self.torch = smc, torch
        self.dev, self.N, self.K, self.V, self.P = dev, N, K, V, P
        self.prompt_base = rank * P
        self.ring = [synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, device=dev,
                                     seed=synth.GEN_SEED_BASE + 2 + 1000 * r + 7 * rank)
                     for r in range(ring)]
        self.logw = synth.uniform_prior(P, N, device=dev)
        total = args.warmup + args.steps + 4
        mk = lambda dt: torch.zeros((total, P, N), dtype=dt, device=dev)
        self.anc, self.off, self.slot = mk(torch.int32), mk(torch.int32), mk(torch.int32)
        self.essrec = torch.zeros((total, P), dtype=torch.float64, device=dev)
        self.out = smc.Outputs(logw=self.logw, status=torch.zeros(P, dtype=torch.int32, device=dev),
                               resampled=torch.zeros(P, dtype=torch.uint8, device=dev),
                               ess=torch.zeros(P, dtype=torch.float64, device=dev),
                               lse=torch.zeros(P, dtype=torch.float64, device=dev),
                               n_ties=torch.zeros(P, dtype=torch.int32, device=dev))
        self.ws = smc.Workspace(dev)
        self.ws.get(P, N, K, V)
        self.kv = None
        if kv:
            L, H, S, d = KV70B["L"], KV70B["H"], KV70B["S"], KV70B["d"]
            self.kv = synth.kv_bits_fast((L, 2, P, N, H, S, d), seed=91 + rank, device=dev)
            self.kv_geom = smc.kv_geometry(self.kv)
            self.Bp = L * 2 * H * S * d * 2
            self.T = 2048
            self.hist = torch.randint(0, V, (P, N, self.T), dtype=torch.int32, device=dev)
            self.hist_geom = dict(n_outer=1, outer_stride=0, prompt_stride=N * self.T * 4,
                                  particle_stride=self.T * 4, seg_count=1, seg_bytes=self.T * 4,
                                  seg_stride=self.T * 4)
        # S8 + S9 in one launch: the 70B KV blocks and the token history share the slot plan
        self.kernels = ["smcsd_step(k_rowstats+k_tail)"] + (["k_kv_reindex(kv+tokens)"] if kv else [])

    def launches_per_step(self):
        return len(self.kernels)

    def kernel_launches_per_step(self):
        """CUDA kernel launches per step: smcsd_step is K1 + K2, the reindex one kernel."""
        return 2 + (1 if self.kv is not None else 0)

    def step(self, i, events=None, inputs=None):
        smc = self.smc
        lp, lq, tok = inputs if inputs is not None else self.ring[i % len(self.ring)]
        o = self.out
        o.ancestors, o.offspring, o.slot_src = self.anc[i], self.off[i], self.slot[i]
        o.ess = self.essrec[i]
        if events: events[0].record()
        smc.smcsd_step(lp, lq, tok, V=self.V, logw_prev=self.logw, eta=math.inf,
                       seed=0x5EED5EED, step=i, prompt_base=self.prompt_base, out=o,
                       fields=(), workspace=self.ws)
        if events: events[1].record()
        if self.kv is not None:
            smc.smcsd_kv_reindex_multi([smc.kv_tensor(self.kv, self.kv, **self.kv_geom),
                                        smc.kv_tensor(self.hist, self.hist, **self.hist_geom)],
                                       self.slot[i])
            if events: events[2].record()

    # algorithmic bytes
    def logit_bytes(self):
        P, N, K, V = self.P, self.N, self.K, self.V
        return P * (2 * N * K * V * 2 + N * K * 4 + 3 * N * 4)

    def kv_bytes(self, steps):
        """Per-step in-place KV + token bytes: (R_src + W_dst) * block, from the recorded plans."""
        off = self.off[steps].cpu()
        kv, tok = [], []
        for s in range(off.shape[0]):
            r = int((off[s] >= 2).sum())
            w = int((off[s] == 0).sum())
            kv.append((r + w) * self.Bp)
            tok.append((r + w) * self.T * 4)
        return kv, tok


def run_ours(args, rank, world, local):
    import torch
    import paper_2604_15672_b200 as smc
    from paper_2604_15672_b200.dist import max_over_ranks

    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    hbm_peak, peak_src = peaks()
    wl = Cfg2Step(dev, rank, args)
    stream = torch.cuda.current_stream(dev)

    # ---- warm-up
    for i in range(args.warmup):
        wl.step(i)
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the launching stream).  The K steps are
    # captured once in a CUDA graph and replayed once (a serving loop replays its step the same
    # way: the binding's ~30 us of host time per call would otherwise pace the ~20 us verify
    # kernels); per-launch timing events are captured with them (external event nodes).
    # The timed graph holds only the steps' kernels (consecutive launches keep their programmatic
    # (PDL) edges); the per-launch breakdown comes from a second graph of the same steps with
    # event nodes between the launches, replayed outside the timed region.
    nk = wl.launches_per_step()
    mk_ev = lambda: torch.cuda.Event(enable_timing=True, external=True)
    ev = [[mk_ev() for _ in range(nk + 1)] for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timing_mode = "cuda_graph"
    graph = graph_ev = None
    try:
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(stream)
        graph, graph_ev = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            with torch.cuda.graph(graph, stream=gs):
                for k in range(args.steps):
                    wl.step(args.warmup + k)
            with torch.cuda.graph(graph_ev, stream=gs):
                for k in range(args.steps):
                    wl.step(args.warmup + k, events=ev[k])
        torch.cuda.synchronize()
    except Exception:                                  # capture unsupported: time the eager loop
        graph = graph_ev = None
        timing_mode = "eager"
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nk + 1)] for _ in range(args.steps)]
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for k in range(args.steps):
                wl.step(args.warmup + k, events=ev[k])
        t1.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    elapsed_ms = t0.elapsed_time(t1)
    if graph is not None:
        del graph
        # (the same steps again, untimed, with the per-launch events)
        graph_ev.replay()
        torch.cuda.synchronize()
        del graph_ev
    per_kernel_ms = [statistics.fmean(ev[k][j].elapsed_time(ev[k][j + 1]) for k in range(args.steps))
                     for j in range(nk)]
    elapsed_ms = max_over_ranks(elapsed_ms, dev)
    ms_per_step = elapsed_ms / args.steps
    value = world * wl.P * args.steps / (elapsed_ms / 1e3)

    # ---- algorithmic bytes and roofline
    timed = list(range(args.warmup, args.warmup + args.steps))
    kvb, tokb = wl.kv_bytes(timed)
    logit_b = wl.logit_bytes()
    kv_avg, tok_avg = statistics.fmean(kvb), statistics.fmean(tokb)
    step_bytes = logit_b + kv_avg + tok_avg
    bytes_by_kernel = [logit_b, kv_avg + tok_avg]
    kernels = []
    traffic = traffic_table()
    for name, ms, b in zip(wl.kernels, per_kernel_ms, bytes_by_kernel):
        gbs = b / (ms / 1e3) / 1e9
        kernels.append({"kernel": name, "avg_ms": round(ms, 5), "algorithmic_bytes": int(b),
                        "achieved_gbs": round(gbs, 1), "frac_of_measured": round(gbs / hbm_peak, 4),
                        "frac_of_8tbs": round(gbs / (NORTH_STAR_TBS * 1e3), 4)})
    dom = max(range(len(kernels)), key=lambda j: per_kernel_ms[j])
    dk = kernels[dom]
    tr = traffic.get(dk["kernel"])
    roofline = {"bound": "hbm", "achieved": dk["achieved_gbs"], "peak": hbm_peak, "unit": "GB/s",
                "frac": round(dk["achieved_gbs"] / hbm_peak, 4),
                "traffic": tr, "kernel": dk["kernel"], "peak_source": peak_src,
                "algorithmic_bytes_per_launch": dk["algorithmic_bytes"]}
    if tr and dk["kernel"] == "k_kv_reindex(kv+tokens)" and wl.off.shape[0] > 3:
        # the ncu capture (scripts/gpu_profile.sh: -k k_kv_reindex -s 3 -c 1 on --warmup 3) is the
        # reindex launch of bench step 3, whose plan (dead slots) differs from the average launch:
        # compare its DRAM bytes with its own algorithmic bytes
        kv3, tok3 = wl.kv_bytes([3])
        alg3 = kv3[0] + tok3[0]
        roofline["traffic_launch"] = {"bench_step": 3, "algorithmic_bytes": int(alg3),
                                      "dram_over_algorithmic": round(tr / alg3, 4) if alg3 else None}
    step_gbs = step_bytes / (ms_per_step / 1e3) / 1e9
    anc = wl.anc[timed].cpu()
    dead = statistics.fmean(float((wl.off[s] == 0).sum()) for s in timed)
    ess_frac = float(wl.essrec[timed].mean().item()) / wl.N

    # ---- end to end through the public API with host buffers (H2D of inputs, D2H of result)
    e2e = run_e2e(wl, args, dev, world)
    secondary, sharded = {}, {}
    if not args.no_secondary:
        del wl.kv
        wl.kv = None
        torch.cuda.empty_cache()
        # Each secondary measurement starts after a short idle (the GPU's power controller caps
        # sustained compute-heavy streams at ~1000 W / ~1620 MHz -- DESIGN.md section 8b) and
        # records the SM clock and clock-event reasons seen during it.
        def settled(fn, *a):
            barrier(world)
            time.sleep(args.settle_s)
            with ClockSampler(dev.index if dev.index is not None else 0) as cs:
                r = fn(*a)
            r["clocks"] = cs.summary()
            return r
        # the sharded configs: cfg4 prompt-sharded (strong scaling over the
        # ranks, steps/s = 1 / max-rank time), cfg5 vocab-sharded TP
        sharded["cfg4"] = settled(measure_cfg4, dev, rank, world, hbm_peak)
        sharded["cfg5"] = settled(measure_cfg5, dev, rank, world, hbm_peak)
        if world == 1:
            secondary["cfg3"] = settled(measure_cfg3, dev, hbm_peak)
            secondary["cfg2_verify"] = settled(measure_cfg2_verify, dev, hbm_peak)
            secondary["powersmc"] = settled(measure_power, dev, hbm_peak)
            secondary["paper_sweep"] = settled(measure_paper_sweep, dev, hbm_peak)

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded LM-like logits, random KV bits; no models)",
        "summary": summarize(per_kernel_ms, sharded, secondary, world),
        "config": {
            "workload": "cfg2: verify+resample V=128256 N=16 K=8 bf16 logits, 1 prompt/GPU "
                        "+ in-place KV reindex of Llama-3.1-70B-shaped KV (80L x 8 KV heads x "
                        "d128 x seq2048 bf16, 640 MiB/particle) + token-history reindex",
            "P_per_gpu": wl.P, "N": wl.N, "K": wl.K, "V": wl.V, "logits_dtype": "bf16",
            "eta": "inf (resample every step)", "parallelism": f"dp{world} (prompts)",
            "timing": timing_mode + " (the K timed steps captured once, replayed once; per-launch "
                      "breakdown from a second replay with event nodes)"
                      if timing_mode == "cuda_graph" else "eager loop",
            "l2": "logits ring of 6 sets (394 MB > 126 MB L2); KV 10.7 GB > L2",
            "kv_mode": "in-place slot plan", "mean_dead_slots": round(dead, 2),
            "mean_ess_over_n": round(ess_frac, 4),
            # chi^2(p_K || q_K) of a K-token block estimated from the realised ESS: ESS/N ->
            # 1 / (1 + chi^2), per drafted token (1 + chi^2_block)^(1/K) - 1
            "chi2_block_est": round(1.0 / ess_frac - 1.0, 4) if ess_frac > 0 else None,
            "chi2_token_est": round((1.0 / ess_frac) ** (1.0 / wl.K) - 1.0, 4) if ess_frac > 0 else None,
        },
        "hbm": {"algorithmic_bytes_per_step": int(step_bytes),
                "achieved_gbs": round(step_gbs, 1),
                "frac_of_measured": round(step_gbs / hbm_peak, 4),
                "frac_of_8tbs": round(step_gbs / (NORTH_STAR_TBS * 1e3), 4)},
        "roofline": roofline,
        "kernels": kernels,
        "breakdown": {"verify_resample_us_event_timed": round(per_kernel_ms[0] * 1e3, 2),
                      "verify_resample_steps_per_s_event_timed": round(1e3 / per_kernel_ms[0], 1),
                      "note": "per-launch times from a second replay of the same steps with event nodes "
                              "between the launches (no PDL overlap across them): the verify part of "
                              "the headline step; the verify path alone under graph replay is "
                              "secondary.cfg2_verify"},
        "e2e": e2e,
        "sharded": sharded,
        "secondary": secondary,
        "gpu_launches": wl.kernel_launches_per_step() * args.steps,
        "clocks": clk.summary(),
        "library": smc.smcsd_version(),
        "ancestor_sample": anc[-1, 0].tolist(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(wl, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)


def summarize(per_kernel_ms, sharded, secondary, world):
    """A short digest near the front of the line (the full objects follow at the end): the
    headline's verify kernel, cfg4 burst / sustained fractions of the measured copy peak, the
    fused TP step, cfg3 and the cfg2 verify path under graph replay."""
    g = lambda d, *ks: _dig(d, ks)
    out = {"n_gpus": world, "headline_verify_us_event_timed": round(per_kernel_ms[0] * 1e3, 2)}
    c4 = sharded.get("cfg4") or {}
    out["cfg4_prompt_steps_per_s"] = c4.get("steps_per_s")
    out["cfg4_frac_burst"] = c4.get("frac_of_measured")
    out["cfg4_frac_sustained"] = g(c4, "sustained", "frac_of_measured")
    out["cfg4_sustained_sm_mhz"] = g(c4, "sustained", "clocks", "sm_mhz")
    c5 = sharded.get("cfg5") or {}
    out["cfg5_tp_ms_per_step"] = c5.get("ms_per_step")
    out["cfg5_tp_path"] = "fused" if "fused_exchange" in c5 and "error" not in c5["fused_exchange"] else (
        "allgather" if c5 else None)
    out["cfg5_tp_overhead_vs_plain"] = g(c5, "fused_exchange", "overhead_vs_plain")
    out["cfg2_verify_graph_us"] = g(secondary, "cfg2_verify", "plain", "graph_us_per_step")
    out["cfg2_verify_graph_frac_of_cold_floor"] = g(secondary, "cfg2_verify", "plain", "graph_frac_of_cold_floor")
    out["cfg3_in_place_frac"] = g(secondary, "cfg3", "in_place", "frac_of_measured")
    return out


def _dig(d, ks):
    for k in ks:
        if not isinstance(d, dict) or k not in d:
            return None
        d = d[k]
    return d


def _time_steps(fn, steps, warmup, world, dev):
    """Device time per step (CUDA events on the current stream), max over ranks."""
    import torch
    from paper_2604_15672_b200.dist import max_over_ranks
    for i in range(warmup):
        fn(i)
    barrier(world)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for i in range(steps):
        fn(warmup + i)
    t1.record()
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(t0.elapsed_time(t1), dev) / steps


def measure_cfg4(dev, rank, world, hbm_peak, steps=20, warmup=3):
    """configs[3]: 64 prompts x N=32 x K=8, V=128256 bf16, prompt-sharded over the ranks
    (strong scaling: 64/G prompts per rank, global prompt index for Philox).  S1-S7 per step
    (the dense KV of 64 x 32 70B particles, 1.3 TB, does not fit: S8 is measured in cfg3)."""
    import torch
    import paper_2604_15672_b200 as smc
    import synth
    from paper_2604_15672_b200.dist import prompt_shard
    P_all, N, K, V = 64, 32, 8, 128256
    b, e = prompt_shard(P_all, world, rank)
    P = e - b
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, device=dev,
                                  seed=synth.GEN_SEED_BASE + 4 + 101 * rank)
    logw = synth.uniform_prior(P, N, device=dev)
    ws = smc.Workspace(dev)
    out = smc.Outputs(logw=logw)
    fn = lambda i: smc.smcsd_step(lp, lq, tok, V=V, logw_prev=logw, eta=math.inf, step=i,
                                  prompt_base=b, out=out, fields=(), workspace=ws)
    ms = _time_steps(fn, steps, warmup, world, dev)
    byts = P * (2 * N * K * V * 2 + N * K * 4 + 3 * N * 4)
    gbs = byts / (ms / 1e3) / 1e9
    # NEXT #2: the same step plus the bonus token (target row K streamed in K1, bonus CTAs)
    fnb = lambda i: smc.smcsd_step(lp, lq, tok, V=V, logw_prev=logw, eta=math.inf, step=i,
                                   prompt_base=b, out=out, fields=(), workspace=ws, bonus=True)
    # sustained: ~3 s of back-to-back steps, the last second timed (the board settles at its
    # 1000 W cap and the SM clock drops), clocks sampled during it
    sustained = None
    if os.environ.get("SMCSD_BENCH_SUSTAINED", "1") == "1":
        t_end = time.time() + 2.0
        i = 0
        while time.time() < t_end:
            fn(i)
            i += 1
            if i % 50 == 0:
                torch.cuda.synchronize(dev)
        with ClockSampler(dev.index if dev.index is not None else 0) as cs:
            ms_sus = _time_steps(fn, max(20, int(1000 / max(ms, 1e-3))), 0, world, dev)
        sustained = {"ms_per_step": round(ms_sus, 4),
                     "frac_of_measured": round(byts / (ms_sus / 1e3) / 1e9 / hbm_peak, 4),
                     "clocks": cs.summary(), "note": "after ~2 s of back-to-back steps (power-capped state)"}
    time.sleep(1.0)                                        # power-state settle (see settled())
    msb = _time_steps(fnb, steps, warmup, world, dev)
    bytb = byts + P * N * V * 2
    gbb = bytb / (msb / 1e3) / 1e9
    del lp, lq, tok
    torch.cuda.empty_cache()
    return {"workload": f"cfg4: {P_all} prompts x N={N} x K={K}, V={V} bf16, {P} prompts/rank, "
                        f"smcsd_step (S1-S7); 8.4 GB/step at G=1 (> L2)",
            "steps_per_s": round(P_all / (ms / 1e3) if world > 1 else P / (ms / 1e3), 1),
            "unit": "prompt-steps/s", "ms_per_step": round(ms, 4), "bytes_per_rank": int(byts),
            "achieved_gbs_per_rank": round(gbs, 1), "frac_of_measured": round(gbs / hbm_peak, 4),
            "frac_of_8tbs": round(gbs / 8000.0, 4),
            "sustained": sustained,
            "with_bonus": {"ms_per_step": round(msb, 4), "bytes_per_rank": int(bytb),
                           "achieved_gbs_per_rank": round(gbb, 1),
                           "frac_of_measured": round(gbb / hbm_peak, 4)}}


def measure_cfg2_verify(dev, hbm_peak, steps=120, warmup=6):
    """cfg2 verification only (smcsd_step S1-S7, no KV), with and without the bonus token
    (NEXT #2): latency per step over a ring of 6 logit sets (394 MB > L2)."""
    import torch
    import paper_2604_15672_b200 as smc
    import synth
    P, N, K, V = 1, 16, 8, 128256
    ring = [synth.lm_logits(P, N, K, V, device=dev, seed=synth.GEN_SEED_BASE + 200 + r) for r in range(6)]
    ws = smc.Workspace(dev)
    out = smc.Outputs()
    res = {"workload": "cfg2 verify: smcsd_step S1-S7, P=1 N=16 K=8 V=128256 bf16, ring of 6 "
                       "(prepared calls: smc.StepPlan)"}
    for bonus in (False, True):
        # a prepared call (smc.StepPlan, ~9 us of host time) so the host does not pace a
        # ~24 us device step; the plain binding call costs ~27 us of host time per step
        plan = smc.StepPlan(*ring[0], V=V, eta=math.inf, out=out, fields=(), workspace=ws, bonus=bonus)
        fn = lambda i, plan=plan: plan.run(*ring[i % 6], step=i)
        ms = _time_steps(fn, steps, warmup, 1, dev)
        byts = 2 * N * K * V * 2 + (N * V * 2 if bonus else 0)
        # SURVEY.md 8(d) protocol: R steps cycling the 6-set ring captured in one CUDA graph,
        # median of 7 replays (no host in the loop).  R = 48: the graph launch (a few us) is
        # spread over 48 steps as in a serving loop; R = 6 (one replay per ring pass, the
        # round-2a protocol) is reported beside it.
        def graph_us(R):
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(torch.cuda.current_stream(dev))
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(gs):
                for i in range(6):
                    smc.smcsd_step(*ring[i], V=V, eta=math.inf, step=i, out=out, fields=(),
                                   workspace=ws, stream=gs, bonus=bonus)
                torch.cuda.synchronize(dev)
                with torch.cuda.graph(graph, stream=gs):
                    for i in range(R):
                        smc.smcsd_step(*ring[i % 6], V=V, eta=math.inf, step=i, out=out, fields=(),
                                       workspace=ws, stream=gs, bonus=bonus)
            graph.replay()
            torch.cuda.synchronize(dev)
            reps = []
            for _ in range(7):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graph.replay()
                e1.record()
                torch.cuda.synchronize(dev)
                reps.append(e0.elapsed_time(e1) / R)
            del graph
            return statistics.median(reps)
        gms = graph_us(48)
        gms6 = graph_us(6)
        res["with_bonus" if bonus else "plain"] = {
            "us_per_step": round(ms * 1e3, 2), "bytes": byts,
            "frac_of_measured": round(byts / (ms / 1e3) / 1e9 / hbm_peak, 4),
            "graph_us_per_step": round(gms * 1e3, 2), "graph_steps_per_replay": 48,
            "graph_us_per_step_r6": round(gms6 * 1e3, 2),
            "graph_frac_of_measured": round(byts / (gms / 1e3) / 1e9 / hbm_peak, 4),
            "graph_frac_of_cold_floor": round(COLD_READ_FLOOR_US * (byts / 65667072) / (gms * 1e3), 4)}
    res["cold_floor_note"] = (f"a cold {65667072 / 1e6:.1f} MB read alone takes {COLD_READ_FLOOR_US} us "
                              "(profiles/r01_ubench_stream.txt, best no-compute stream), above the "
                              "11.73 us that 70% of 8 TB/s would need: the 70% bar is out of reach "
                              "for a single cold cfg2 prompt; the fraction of that floor is reported")
    del ring
    torch.cuda.empty_cache()
    return res


PAPER_NK = [(12, 8), (8, 16), (6, 12), (12, 16), (4, 32), (8, 32), (4, 64), (16, 12), (8, 48), (8, 8),
            (4, 16), (8, 26)]


def measure_paper_sweep(dev, hbm_peak, replays=5):
    """The paper's batch-1..16 operating points: (N, K) from PAPER.md:537-674, P from
    PAPER.md:729, V = 128256 bf16, smcsd_step S1-S7 (eta = inf).  Each point: R = max(24, ring)
    steps cycling a ring of logit sets larger than 3x L2 (>= 2 sets, <= 16) captured in one CUDA
    graph, median of `replays` replays (no host in the loop; cold inputs; the graph launch spread
    over R steps); the fraction is of the measured copy peak for the algorithmic logit bytes
    2 N K V 2 P."""
    import torch
    import paper_2604_15672_b200 as smc
    import synth
    V = 128256
    rows = []
    for P in (1, 4, 8, 16):
        for N, K in PAPER_NK:
            byts = 2 * N * K * V * 2 * P
            nring = max(2, min(16, -(-3 * 126 * 2 ** 20 // byts)))
            R = max(24, nring)
            ring = [synth.lm_logits(P, N, K, V, device=dev, seed=31 + r) for r in range(nring)]
            ws, out = smc.Workspace(dev), smc.Outputs()
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(torch.cuda.current_stream(dev))
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(gs):
                for i in range(nring):
                    smc.smcsd_step(*ring[i], V=V, eta=math.inf, step=i, out=out, fields=(),
                                   workspace=ws, stream=gs)
                torch.cuda.synchronize(dev)
                with torch.cuda.graph(graph, stream=gs):
                    for i in range(R):
                        smc.smcsd_step(*ring[i % nring], V=V, eta=math.inf, step=i, out=out, fields=(),
                                       workspace=ws, stream=gs)
            graph.replay()
            torch.cuda.synchronize(dev)
            reps = []
            for _ in range(replays):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graph.replay()
                e1.record()
                torch.cuda.synchronize(dev)
                reps.append(e0.elapsed_time(e1) / R)
            ms = statistics.median(reps)
            rows.append([N, K, P, round(ms * 1e3, 2), round(byts / (ms / 1e3) / 1e9 / hbm_peak, 3)])
            del graph, ring
            torch.cuda.empty_cache()
    return {"workload": "paper operating points (PAPER.md:537-674, 729): smcsd_step S1-S7, V=128256 bf16, "
                        "CUDA graph of max(24, ring) steps over a ring > 3x L2 (cold inputs), median of 5",
            "columns": ["N", "K", "P", "us_per_step", "frac_of_measured"], "rows": rows}


def measure_power(dev, hbm_peak, steps=20, warmup=3):
    """NEXT #4 PowerSMC (App. F): K = 1, one model, log w = ln sum_v p_v^alpha per particle,
    then S4; 64 prompts x N = 32, V = 128256 bf16 (525 MB).  alpha = 4 (integer: the power
    sum reuses the ex2 of the softmax sum) and alpha = 2.5 (a second ex2 per element)."""
    import torch
    import paper_2604_15672_b200 as smc
    import synth
    P, N, V = 64, 32, 128256
    lg, _, _ = synth.lm_logits(P, N, 1, V, dtype=torch.bfloat16, device=dev, bonus=False,
                               seed=synth.GEN_SEED_BASE + 44)
    ws = smc.Workspace(dev)
    out = smc.Outputs()
    res = {"workload": f"PowerSMC weights: {P} prompts x N={N}, V={V} bf16 (K=1, no bonus)"}
    byts = P * N * V * 2
    for a in (4.0, 2.5):
        fn = lambda i: smc.smcsd_powersmc_weights(lg, V=V, alpha=a, out=out, workspace=ws)
        ms = _time_steps(fn, steps, warmup, 1, dev)
        gbs = byts / (ms / 1e3) / 1e9
        res[f"alpha_{a}"] = {"ms_per_step": round(ms, 4), "achieved_gbs": round(gbs, 1),
                             "frac_of_measured": round(gbs / hbm_peak, 4)}
    del lg
    torch.cuda.empty_cache()
    return res


def measure_cfg5(dev, rank, world, hbm_peak, steps=20, warmup=3):
    """configs[4]: V=128256 vocab-sharded over the ranks (TP), P=1, N=64, K=8 bf16.  A step is
    smcsd_weights_partial on this rank's columns -> all_gather of 16 B per row (S10, NCCL) ->
    smcsd_weights_combine (rank-order merge: identical on every rank) -> smcsd_resample (same
    Philox counter everywhere, no communication).  At one GPU the shard is the whole row."""
    import torch
    import paper_2604_15672_b200 as smc
    import synth
    from paper_2604_15672_b200.dist import exchange_partials_into, vocab_shard
    P, N, K, V = 1, 64, 8, 128256
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, device=dev,
                                  seed=synth.GEN_SEED_BASE + 5)   # same on every rank
    b, e = vocab_shard(V, world, rank)
    w = e - b
    ldw = synth.padded_ld(w, torch.bfloat16)
    sp = torch.zeros((P, N, K + 1, ldw), dtype=torch.bfloat16, device=dev)
    sq = torch.zeros((P, N, K, ldw), dtype=torch.bfloat16, device=dev)
    sp[..., :w] = lp[..., b:e]
    sq[..., :w] = lq[..., b:e]
    del lp, lq
    torch.cuda.empty_cache()
    ws_p, ws_c = smc.Workspace(dev), smc.Workspace(dev)
    part = torch.empty((P, 2, N, K, 4), dtype=torch.float32, device=dev)
    gathered = torch.empty((world, P, 2, N, K, 4), dtype=torch.float32, device=dev)
    logw = synth.uniform_prior(P, N, device=dev)
    oc = smc.Outputs(logw=torch.empty_like(logw))
    orr = smc.Outputs(logw=logw)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    phases = [0.0, 0.0, 0.0]

    def fn(i, ev=None):
        if ev: ev[0].record()
        smc.smcsd_weights_partial(sp, sq, tok, v_begin=b, v_len=w, partials=part, workspace=ws_p)
        if ev: ev[1].record()
        if world > 1:
            exchange_partials_into(gathered, part)
        else:
            gathered[0].copy_(part)
        if ev: ev[2].record()
        smc.smcsd_weights_combine(gathered, tok, V=V, logw_prev=logw, out=oc, fields=(), workspace=ws_c)
        smc.smcsd_resample(oc.logw, eta=math.inf, step=i, out=orr, fields=())
        if ev: ev[3].record()
    ms = _time_steps(fn, steps, warmup, world, dev)        # overlapped steps: the metric
    for i in range(steps):                                 # phase breakdown (events per phase)
        fn(i, ev)
        torch.cuda.synchronize()
        for j in range(3):
            phases[j] += ev[j].elapsed_time(ev[j + 1])
    byts = 2 * N * K * w * 2
    part_ms = phases[0] / steps
    gbs = byts / (part_ms / 1e3) / 1e9
    res = {"workload": f"cfg5: P=1, N={N}, K={K}, V={V} bf16 vocab-sharded {world}-way "
                       f"({w} columns on this rank); product path smcsd_tp_step (S10 fused into "
                       f"K1 over peer memory); NCCL all-gather / all-reduce forms as baselines",
           "bytes_per_rank": int(byts),
           "allgather_exchange": {
               "ms_per_step": round(ms, 4), "steps_per_s": round(1e3 / ms, 1),
               "path": "partial -> all_gather -> combine -> resample",
               "note": "phase times below are measured with a host sync per step (not overlapped)",
               "partial_ms": round(part_ms, 4), "exchange_ms": round(phases[1] / steps, 4),
               "combine_resample_ms": round(phases[2] / steps, 4),
               "partial_achieved_gbs": round(gbs, 1), "partial_frac_of_measured": round(gbs / hbm_peak, 4)}}
    # S10 in the north star's all-reduce form: all_reduce(MAX) of {m, x}, smcsd_partials_rescale,
    # all_reduce(SUM) of the rescaled sums, combine with G = 1
    from paper_2604_15672_b200.dist import exchange_partials_allreduce
    oa = smc.Outputs(logw=torch.empty_like(logw))

    def fna(i):
        smc.smcsd_weights_partial(sp, sq, tok, v_begin=b, v_len=w, partials=part, workspace=ws_p)
        if world > 1:
            merged = exchange_partials_allreduce(part)
        else:
            merged = smc.smcsd_partials_rescale(part, part.clone()).unsqueeze(0)
        smc.smcsd_weights_combine(merged, tok, V=V, logw_prev=logw, out=oa, fields=(), workspace=ws_c)
        smc.smcsd_resample(oa.logw, eta=math.inf, step=i, out=orr, fields=())
    msa = _time_steps(fna, steps, warmup, world, dev)
    res["allreduce_exchange"] = {"ms_per_step": round(msa, 4), "steps_per_s": round(1e3 / msa, 1),
                                 "path": "partial -> all_reduce(MAX) -> smcsd_partials_rescale -> "
                                         "all_reduce(SUM) -> combine (G = 1) -> resample"}
    # S10 fused into K1 (smcsd_tp_step): partials pushed to every rank's exchange buffer over
    # peer memory, epoch flags, tail merges in rank order -- 2 launches, no collective call
    cpu_group = None
    if world > 1:
        import torch.distributed as tdist
        cpu_group = tdist.new_group(backend="gloo")        # error agreement off the GPU
    try:
        from paper_2604_15672_b200.dist import TPExchange
        ex = TPExchange(P, N, K, V) if world > 1 else TPExchange.local_group(P, N, K, V, 1, device=dev)[0]
        of = smc.Outputs(logw=logw)
        wsf = smc.Workspace(dev)
        fnf = lambda i: ex.step(sp, sq, tok, logw_prev=logw, eta=math.inf, step=i, out=of,
                                fields=(), workspace=wsf)
        # one checked step first: a peer mapping that does not work shows up as ST_EXCHANGE
        # after the bounded wait (20 s), never as a hang; then the path is not timed.  The
        # ranks agree over a CPU (gloo) group, which still works if one rank's CUDA context
        # faulted, so every rank skips the timing together.
        bad = 0.0
        try:
            fnf(0)
            torch.cuda.synchronize()
            bad = float((of.status != 0).any().item())
        except Exception:
            bad = 1.0
        if world > 1:
            import torch.distributed as tdist
            t = torch.tensor([bad])
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX, group=cpu_group)
            bad = float(t.item())
        if bad != 0:
            raise RuntimeError(f"fused exchange check failed on some rank (this rank: {bad})")
        msf = _time_steps(fnf, steps, warmup, world, dev)
        torch.cuda.synchronize()
        # the shard's K1 (+ row merge) alone, timed the same way (no host sync between steps)
        fnp_ = lambda i: smc.smcsd_weights_partial(sp, sq, tok, v_begin=b, v_len=w, partials=part,
                                                   workspace=ws_p)
        ms_k1 = _time_steps(fnp_, steps, warmup, world, dev)
        res["fused_exchange"] = {"ms_per_step": round(msf, 4), "steps_per_s": round(1e3 / msf, 1),
                                 "status_ok": bool((of.status == 0).all().item()),
                                 # the two launches of one call cannot be split by events: the
                                 # shard's K1 (+ merge) timed alone as smcsd_weights_partial, the
                                 # rest is the push / flag exchange + S2-S7 tail
                                 "breakdown": {"k1_shard_ms": round(ms_k1, 4),
                                               "exchange_plus_tail_ms": round(msf - ms_k1, 4),
                                               "note": "k1_shard_ms: smcsd_weights_partial on the "
                                                       "same shard timed alone (K1 + row merge)"},
                                 "path": "smcsd_tp_step: K1 pushes each partial to every rank as "
                                         "two tagged 8-byte words (P2P relaxed stores, no fence or "
                                         "flag); the tail polls them + S2-S7"}
        if world == 1:
            # one rank holds the whole vocabulary: the plain smcsd_step on the same inputs, so
            # the line shows what the fused exchange costs (profiles/r02k_tp_overhead_decomposition.txt)
            op, wsq = smc.Outputs(logw=logw), smc.Workspace(dev)
            fnq = lambda i: smc.smcsd_step(sp, sq, tok, V=V, logw_prev=logw, eta=math.inf, step=i,
                                           out=op, fields=(), workspace=wsq)
            msq = _time_steps(fnq, steps, warmup, world, dev)
            res["fused_exchange"]["plain_step_ms"] = round(msq, 4)
            res["fused_exchange"]["overhead_vs_plain"] = round(msf / msq - 1.0, 4)
        # the product path is the line's cfg5 figure
        res["ms_per_step"] = round(msf, 4)
        res["steps_per_s"] = round(1e3 / msf, 1)
        res["achieved_gbs_per_rank"] = round(byts / (msf / 1e3) / 1e9, 1)
        res["frac_of_measured"] = round(byts / (msf / 1e3) / 1e9 / hbm_peak, 4)
        ex.close()
    except Exception as exc:  # pragma: no cover - reported, never fatal for the bench
        res["fused_exchange"] = {"error": repr(exc)[:300]}
        res["ms_per_step"] = round(ms, 4)                  # fall back to the NCCL all-gather form
        res["steps_per_s"] = round(1e3 / ms, 1)
        res["path_timed"] = "allgather_exchange (fused exchange failed)"
    return res


def measure_cfg3(dev, hbm_peak, steps=5, warmup=2):
    """configs[2]: Llama-3.1-70B KV (80 L x 2 x 8 heads x 2048 x 128 bf16 = 640 MiB/particle),
    N=32, pinned ancestor pattern (lam = 0 on even n, -inf on odd n: 16 sources x 2 offspring).
    One step = smcsd_resample + smcsd_kv_reindex, out of place and in place."""
    import torch
    import paper_2604_15672_b200 as smc
    import synth
    N = 32
    L, H, S, d = KV70B["L"], KV70B["H"], KV70B["S"], KV70B["d"]
    lw = torch.zeros((1, N), device=dev)
    lw[0, 1::2] = -float("inf")
    res = {}
    Bp = L * 2 * H * S * d * 2
    src = synth.kv_bits_fast((L, 2, 1, N, H, S, d), seed=7, device=dev)
    geom = smc.kv_geometry(src)
    dst = torch.empty_like(src)
    o = smc.smcsd_resample(lw.clone(), eta=math.inf)
    torch.cuda.synchronize()
    off = o.offspring[0].cpu()
    distinct, dead = int((off >= 1).sum()), int((off == 0).sum())
    multi = int((off >= 2).sum())
    for mode in ("out_of_place", "in_place"):
        lwb = lw.clone()

        def fn(i, mode=mode):
            lwb.copy_(lw)
            r = smc.smcsd_resample(lwb, eta=math.inf, step=i, out=o)
            if mode == "out_of_place":
                smc.smcsd_kv_reindex(dst, src, r.ancestors, **geom)
            else:
                smc.smcsd_kv_reindex(src, src, r.slot_src, **geom)
        ms = _time_steps(fn, steps, warmup, 1, dev)
        byts = ((distinct + N) if mode == "out_of_place" else (multi + dead)) * Bp
        gbs = byts / (ms / 1e3) / 1e9
        res[mode] = {"steps_per_s": round(1e3 / ms, 2), "ms_per_step": round(ms, 4),
                     "algorithmic_bytes": int(byts), "achieved_gbs": round(gbs, 1),
                     "frac_of_measured": round(gbs / hbm_peak, 4), "frac_of_8tbs": round(gbs / 8000.0, 4)}
    del src, dst
    torch.cuda.empty_cache()
    # NEXT #1, the paper's mechanism: the same ancestors applied to block tables
    # (16-token pages: 128 per particle, the first 8 = shared prompt pages) + refcounts; no KV
    # content moves.  Tables double-buffered (swapped every step).
    PG, shared = S // 16, 8
    tab = torch.full((1, N, PG), -1, dtype=torch.int32, device=dev)
    ids = torch.arange(shared, dtype=torch.int32, device=dev)
    own = shared + torch.arange(N * (PG - shared), dtype=torch.int32, device=dev).view(N, PG - shared)
    tab[0, :, :shared] = ids
    tab[0, :, shared:] = own
    npg = torch.full((1, N), PG, dtype=torch.int32, device=dev)
    num_pages = shared + N * (PG - shared)
    refc = torch.ones(num_pages, dtype=torch.int32, device=dev)
    refc[:shared] = N
    freed = torch.zeros(num_pages, dtype=torch.uint8, device=dev)
    bufs = [(tab, npg), (torch.empty_like(tab), torch.empty_like(npg))]
    lwb = lw.clone()

    def fnp(i):
        lwb.copy_(lw)
        r = smc.smcsd_resample(lwb, eta=math.inf, step=i, out=o)
        (ts, ns), (td, nd) = bufs[i % 2], bufs[(i + 1) % 2]
        smc.smcsd_kv_reindex_paged(ts, ns, refc, r.ancestors, table_dst=td, n_pages_dst=nd, freed=freed)
    msp = _time_steps(fnp, 20, 3, 1, dev)
    res["paged"] = {"us_per_step": round(msp * 1e3, 2), "kv_content_bytes": 0,
                    "table_bytes": int(2 * N * PG * 4 + num_pages * 5),
                    "vs_dense_in_place": round(res["in_place"]["ms_per_step"] / msp, 1),
                    "note": "resample + block-table/refcount reindex (K5); pages of 16 tokens"}
    res["paged_round"] = measure_paged_round(dev, hbm_peak)
    res["workload"] = ("cfg3: 70B KV, N=32, pinned pattern (16 sources x 2 offspring, 16 dead slots); "
                       "step = smcsd_resample + smcsd_kv_reindex (dense) or smcsd_kv_reindex_paged")
    return res


def measure_paged_round(dev, hbm_peak, rounds=12, warmup=3):
    """One engine round on the paper's pointer mechanism at the 70B KV shape:
    resample (N=32, pinned pattern: 16 sources x 2) -> paged reindex (block tables + refcounts)
    -> paged append of K+1 = 9 tokens per particle with copy-on-write of the shared partial tail
    pages (smcsd_kv_append_paged).  The pool holds every page of the 80 layers x {K, V} (8 KV
    heads x d 128 bf16, 16-token pages): the copy-on-write moves only the filled tokens of the
    copied tails.  Each round starts from the same state (tables restored by a device copy)."""
    import torch
    import paper_2604_15672_b200 as smc
    N, page, K1 = 32, 16, 9
    L, H, S, d = KV70B["L"], KV70B["H"], KV70B["S"], KV70B["d"]
    seq0 = S - K1 - 3                                 # 2036 tokens: a 4-token partial tail page
    PG = (S + page - 1) // page + 1
    own = (seq0 + page - 1) // page
    num_pages = N * own + N * 2 + 64
    pool = torch.empty((L * 2, num_pages, page, H, d), dtype=torch.bfloat16, device=dev)
    pool.view(torch.int16).random_(-32768, 32767)
    geom = smc.paged_pool_geometry(pool)
    tab0 = torch.full((1, N, PG), -1, dtype=torch.int32, device=dev)
    tab0[0, :, :own] = torch.arange(N * own, dtype=torch.int32, device=dev).view(N, own)
    npg0 = torch.full((1, N), own, dtype=torch.int32, device=dev)
    sl0 = torch.full((1, N), seq0, dtype=torch.int32, device=dev)
    rc0 = torch.zeros(num_pages, dtype=torch.int32, device=dev)
    rc0[:N * own] = 1
    lw = torch.zeros((1, N), device=dev)
    lw[0, 1::2] = -float("inf")
    tab, npg, sl, rc = tab0.clone(), npg0.clone(), sl0.clone(), rc0.clone()
    tab2, npg2 = torch.empty_like(tab), torch.empty_like(npg)
    nn = torch.full((1, N), K1, dtype=torch.int32, device=dev)
    o = smc.Outputs()
    ao = smc.AppendOutputs()
    pools = (smc.kv_pool(pool, **geom),)

    def reset():
        tab.copy_(tab0); npg.copy_(npg0); sl.copy_(sl0); rc.copy_(rc0)

    def round_(i):
        r = smc.smcsd_resample(lw, eta=math.inf, step=i, out=o)
        smc.smcsd_kv_reindex_paged(tab, npg, rc, r.ancestors, table_dst=tab2, n_pages_dst=npg2)
        sl.copy_(torch.gather(sl, 1, r.ancestors.long()))
        smc.smcsd_kv_append_paged(tab2, npg2, sl, rc, nn, page_size=page, max_new=K1, pools=pools, out=ao)

    for i in range(warmup):
        reset(); round_(i)
    torch.cuda.synchronize()
    copies = int((ao.cow_dst >= 0).sum().item())
    tokens = int(ao.cow_tokens.sum().item())
    ok = int(ao.result.item()) == 0
    # a serving loop replays the round from a CUDA graph (the binding's host time per call would
    # pace it otherwise): graph(reset + round) - graph(reset), median of `rounds` replays each
    gs = torch.cuda.Stream(dev)
    gs.wait_stream(torch.cuda.current_stream(dev))
    g_full, g_reset = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        reset(); round_(0)
        torch.cuda.synchronize(dev)
        with torch.cuda.graph(g_full, stream=gs):
            reset(); round_(0)
        with torch.cuda.graph(g_reset, stream=gs):
            reset()

    def med(g):
        ts = []
        for _ in range(rounds):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize(dev)
            ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)
    ms = max(med(g_full) - med(g_reset), 0.0)
    del g_full, g_reset
    cow_bytes = tokens * H * d * 2 * L * 2
    del pool
    torch.cuda.empty_cache()
    return {"us_per_round": round(ms * 1e3, 2), "ok": ok, "cow_pages": copies,
            "cow_content_bytes": int(cow_bytes), "resample_content_bytes": 0,
            "dense_equivalent_bytes_in_place": int(2 * 16 * L * 2 * H * S * d * 2),
            "note": "resample + smcsd_kv_reindex_paged + smcsd_kv_append_paged (K+1 = 9 tokens, "
                    "copy-on-write of shared 4-token tails) over a 70B-shaped paged pool; "
                    "CUDA-graph replay from the same start state, minus the replayed state reset"}


def run_e2e(wl, args, dev, world):
    """Same metric through smcsd_step / smcsd_kv_reindex_multi with inputs from pinned host
    memory: every step copies that step's logits + tokens + prior H2D and reads logw +
    ancestors D2H.  The H2D copies run on a copy stream into two alternating device buffers,
    so step i+1's inputs cross PCIe while step i's kernels run (a serving loop prefetches the
    next batch the same way); every copy of every step is inside the timed region."""
    import torch
    host = [(lp.cpu().pin_memory(), lq.cpu().pin_memory(), tok.cpu().pin_memory())
            for lp, lq, tok in wl.ring[:2]]
    stages = [[torch.empty_like(t) for t in wl.ring[0]] for _ in range(2)]
    prior_h = wl.logw.cpu().pin_memory()
    res_w = torch.empty_like(prior_h).pin_memory()
    res_a = torch.empty((wl.P, wl.N), dtype=torch.int32).pin_memory()
    steps = max(3, min(args.steps, 50))
    base = args.warmup + args.steps
    comp = torch.cuda.current_stream(dev)
    n_copy = int(os.environ.get("SMCSD_E2E_COPY_STREAMS", "1"))
    copies = [torch.cuda.Stream(dev) for _ in range(n_copy)]    # one copy engine each
    h2d_done = [[torch.cuda.Event() for _ in range(n_copy)] for _ in range(2)]
    used = [torch.cuda.Event() for _ in range(2)]

    def h2d(i):
        b = i % 2
        for k, cs in enumerate(copies):                       # lp | lq + tokens
            cs.wait_event(used[b])                            # buffer b free again
            with torch.cuda.stream(cs):
                for j, (s_, t) in enumerate(zip(stages[b], host[i % len(host)])):
                    if min(j, n_copy - 1) == k:
                        s_.copy_(t, non_blocking=True)
                h2d_done[b][k].record(cs)

    def compute(i):
        b = i % 2
        for ev in h2d_done[b]:
            comp.wait_event(ev)
        wl.logw.copy_(prior_h, non_blocking=True)
        wl.step(base + (i % 4), inputs=stages[b])
        used[b].record(comp)
        res_w.copy_(wl.logw, non_blocking=True)
        res_a.copy_(wl.anc[base + (i % 4)], non_blocking=True)

    def run(n, t_start=None):
        if t_start is not None:
            for cs in copies:
                cs.wait_event(t_start)                        # step 0's copy inside the region
        h2d(0)
        for i in range(n):
            if i + 1 < n:
                h2d(i + 1)
            compute(i)

    run(2)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    t0.record(comp)
    run(steps, t0)
    t1.record(comp)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    from paper_2604_15672_b200.dist import max_over_ranks
    ms = max_over_ranks(t0.elapsed_time(t1), dev)
    h2d_b = sum(t.numel() * t.element_size() for t in host[0]) + prior_h.numel() * 4
    d2h = res_w.numel() * 4 + res_a.numel() * 4
    # the PCIe bound: the same H2D copies alone, back to back on the copy stream(s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(comp)
    for i in range(steps):
        for cs in copies:
            cs.wait_event(e0)
        h2d(i)
    for b_ in range(2):
        for ev in h2d_done[b_]:
            comp.wait_event(ev)
    e1.record(comp)
    torch.cuda.synchronize()
    ms_copy = max_over_ranks(e0.elapsed_time(e1), dev)
    return {"value": round(world * wl.P * steps / (ms / 1e3), 3), "unit": "steps/s",
            "h2d_bytes_per_step": int(h2d_b), "d2h_bytes_per_step": int(d2h),
            "steps": steps, "wall_s": round(wall, 4),
            "h2d_gbs": round(h2d_b * steps / (ms / 1e3) / 1e9, 2),
            "h2d_copy_alone_gbs": round(h2d_b * steps / (ms_copy / 1e3) / 1e9, 2),
            "note": f"inputs H2D on {n_copy} copy stream(s), double-buffered (step i+1's copy "
                    "overlaps step i)"}


# ------------------------------------------------------------------------------ CPU legs
def oracle_step_sample(N=16, K=8, V=128256, kv_layers=1, seed=None, logits=None):
    """One bounded sample of the cfg2 step on the host with the oracle: full S1-S7 on one
    prompt's logits, plus the in-place KV reindex of `kv_layers` of the 80 layers (scaled).
    Returns (seconds for S1-S7, seconds for the KV sample, scale factor for the KV)."""
    import numpy as np
    import torch
    import oracle
    import synth
    if logits is None:
        lp, lq, tok = synth.lm_logits(1, N, K, V, dtype=torch.bfloat16,
                                      seed=seed or synth.GEN_SEED_BASE + 2)
        logits = (lp.view(torch.int16).numpy().view(np.uint16),
                  lq.view(torch.int16).numpy().view(np.uint16), tok.numpy())
    lp, lq, tok = logits
    prior = np.full((1, N), np.float32(-math.log(N)), np.float32)
    t0 = time.perf_counter()
    w = oracle.weights(lp, lq, tok, V=V, logw_prev=prior)
    r = oracle.resample(w["logw"], eta=math.inf, seed=0x5EED5EED, step=0)
    t1 = time.perf_counter()
    H, S, d = KV70B["H"], KV70B["S"], KV70B["d"]
    kv = np.empty((kv_layers, 2, 1, N, H, S, d), np.int16)
    kv.view(np.uint8)[...] = 7
    geom = dict(n_outer=kv_layers * 2, outer_stride=N * H * S * d * 2, prompt_stride=N * H * S * d * 2,
                particle_stride=H * S * d * 2, seg_count=H, seg_bytes=S * d * 2, seg_stride=S * d * 2)
    t2 = time.perf_counter()
    oracle.kv_reindex(kv, kv, r["slot_src"], **geom)
    t3 = time.perf_counter()
    return t1 - t0, t3 - t2, KV70B["L"] / kv_layers, logits


def host_cpu():
    """(model name, usable cores) of this host (the GPU box's, when run there)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except Exception:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
    return model, cores


def cpu_baseline(wl, budget_s=12.0):
    """The oracle as it stands on this host, on a bounded sample: single-threaded (liboracle.so)
    and on all usable cores (liboracle_omp.so: the same source with OpenMP over the rows of
    S1+S2 and the KV copy planes; bit-identical outputs)."""
    import numpy as np
    import torch
    import oracle
    lp, lq, tok = wl.ring[0]
    logits = (lp.cpu().view(torch.int16).numpy().view(np.uint16),
              lq.cpu().view(torch.int16).numpy().view(np.uint16), tok.cpu().numpy())
    model, cores = host_cpu()
    res = {}
    for threads in sorted({1, cores}):
        used = oracle.set_threads(threads)
        reps, t_w, t_kv = 0, [], []
        start = time.perf_counter()
        scale = 80.0
        while reps < 1 or (time.perf_counter() - start < budget_s / 2 and reps < 20):
            a, b, scale, logits = oracle_step_sample(logits=logits, kv_layers=2)
            t_w.append(a); t_kv.append(b)
            reps += 1
        step_s = statistics.fmean(t_w) + statistics.fmean(t_kv) * scale
        res[threads] = dict(value=round(1.0 / step_s, 4), cores=used, reps=reps,
                            s1_s7_s=round(statistics.fmean(t_w), 4),
                            kv_per_layer_s=round(statistics.fmean(t_kv) / 2, 5))
    oracle.set_threads(1)
    best = res[max(res)]
    return {"value": best["value"], "unit": "steps/s", "cores": best["cores"], "kind": "oracle",
            "sample": f"{best['reps']} x (full S1-S7 of one cfg2 prompt, 256 rows x 128256 bf16; "
                      f"+ in-place KV reindex of 2 of 80 layers, scaled x80)",
            "single_thread": {**res[1], "unit": "steps/s"},
            "all_cores": {**best, "unit": "steps/s"},
            "cpu_model": model, "host_cores_available": cores}


def run_reference(args, rank, world):
    """--impl reference: the oracle, as it stands, on this host's cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    model, cores = host_cpu()
    used = oracle.set_threads(cores)             # the box's host cores (OpenMP timing build)
    t_steps = []
    logits = None
    for i in range(args.warmup + args.steps):
        a, b, scale, logits = oracle_step_sample(logits=logits, kv_layers=1)
        if i >= args.warmup:
            t_steps.append(a + b * scale)
    step_s = statistics.fmean(t_steps)
    value = 1.0 / step_s
    line = {"metric": METRIC, "impl": "reference", "value": round(value, 4), "unit": "steps/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(step_s * 1e3, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg2 (see ours); oracle: full S1-S7 per step + 1 of 80 KV "
                                   "layers reindexed and scaled x80",
                       "P_per_gpu": 1, "N": 16, "K": 8, "V": 128256},
            "cpu_baseline": {"value": round(value, 4), "unit": "steps/s", "cores": used,
                             "kind": "oracle", "cpu_model": model,
                             "sample": "per step: S1-S7 of one cfg2 prompt + KV reindex of 1 "
                                       "layer of 80 (scaled); OpenMP over the S1+S2 rows"},
            "e2e": {"value": round(value, 4), "unit": "steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args) -> int:
    """`python bench.py --gpus N` (N > 1) without a torchrun wrapper: launch N ranks of this
    script the way the driver does (torch.distributed.run, one process per GPU, rendezvous on
    127.0.0.1), forward stdout/stderr, and return the launcher's exit code."""
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cfg2", choices=["cfg2"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--settle-s", type=float, default=1.0,
                    help="idle seconds before each secondary measurement (power-state settle)")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg3/cfg4 measurements")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        ap.error(f"--gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}: launch one "
                 "rank per GPU (torchrun --nproc-per-node N ... --gpus N)")
    rank, world, local = dist_env(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
