"""GPU: the tail variants of smcsd_step / smcsd_weights against each other (bit-identical outputs)
and against the CPU oracle (staged protocol: the oracle's S4-S7 from the GPU's logw_pre gives the
same ancestry):
  * the small polling cluster tail k_tail_small (smcsd_tail_small.cuh, default for small steps),
  * the 256-thread polling tail (smcsd_set_small_tail(0)),
  * the wait-for-K1 tail (smcsd_set_poll_tail(0)).
Each runs twice on one workspace: the polling tails leave K1's word array zero for the next call."""
import math

import numpy as np
import pytest
import torch

import synth
from gpu_util import max_abs, np_, to_host

pytestmark = pytest.mark.gpu

FIELDS = ("logw", "logw_pre", "logp_tok", "logq_tok", "lse", "ess", "wnorm", "status", "ancestors",
          "offspring", "slot_src", "resampled", "n_ties")


@pytest.fixture(scope="module")
def smc():
    import paper_2604_15672_b200 as m
    assert torch.cuda.is_available()
    yield m
    _set(m, "small")


def _bits(t):
    return t.view(torch.uint8) if t.is_floating_point() else t


def _set(smc, variant):
    smc.smcsd_set_poll_tail(variant != "wait")
    smc.smcsd_set_small_tail(variant not in ("wait", "poll256"))


def _run(smc, lt, mode, lp, lq, tok, ws, **kw):
    _set(smc, lt)
    try:
        if mode == "step":
            o = smc.smcsd_step(lp, lq, tok, workspace=ws, **kw)
        else:
            kw = {k: v for k, v in kw.items() if k in ("V", "n_drafted", "logw_prev", "alpha", "inv_temp_p")}
            o = smc.smcsd_weights(lp, lq, tok, workspace=ws, **kw)
        torch.cuda.synchronize()
    finally:
        _set(smc, "small")
    return {f: getattr(o, f).clone() for f in FIELDS if getattr(o, f, None) is not None}


@pytest.mark.parametrize("P,N,K,V,dtype,extra", [
    (1, 16, 8, 128256, torch.bfloat16, {}),                                  # cfg2
    (1, 4, 4, 1000, torch.float32, {}),                                      # one pass, cfg1-like
    (3, 32, 8, 50001, torch.bfloat16, {}),                                   # 4 passes, ragged V
    (2, 7, 3, 20001, torch.float32, {"scheme": 1}),                          # multinomial
    (1, 1, 1, 7, torch.float32, {}),                                         # N = 1, V < vector
    (4, 32, 16, 128256, torch.bfloat16, {"eta": None}),                      # eta = N/2, 1024 rows
    (2, 12, 8, 131072, torch.bfloat16, {}),                                  # 16 full segments
    (5, 8, 16, 32000, torch.bfloat16, {"alpha": 0.7, "inv_temp_p": 1.3}),
    (2, 32, 2, 60000, torch.bfloat16, {}),                                   # 4 small CTAs, K = 2
    (1, 3, 5, 9000, torch.float32, {}),                                      # K = 5: S3 in the finisher
    (2, 6, 12, 30000, torch.bfloat16, {}),                                   # K = 12: S3 in the finisher
    (1, 8, 32, 50000, torch.bfloat16, {"scheme": 1}),                        # K = 32: 16 small CTAs
    (1, 64, 8, 128256, torch.bfloat16, {}),                                  # N = 64: 2 lanes per row
    (2, 40, 6, 30000, torch.float32, {"scheme": 1}),                         # S3 in the finisher, N > 32
    (1, 48, 8, 20000, torch.bfloat16, {"eta": None}),
])
@pytest.mark.parametrize("mode", ["step", "weights"])
def test_tail_variants_bit_identical(smc, P, N, K, V, dtype, extra, mode):
    dev = torch.device("cuda")
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=dtype, seed=900 + N + V, bonus=False)
    lp, lq, tok = lp.to(dev), lq.to(dev), tok.to(dev)
    g = torch.Generator().manual_seed(N * 7 + K)
    nd = torch.randint(0, K + 1, (P, N), dtype=torch.int32, generator=g).to(dev)
    prev = (torch.randn(P, N, generator=g) * 0.3).to(dev)
    for ndv in (None, nd):
        kw = dict(V=V, n_drafted=ndv, logw_prev=prev, step=3, eta=extra.get("eta", math.inf))
        kw.update({k: v for k, v in extra.items() if k != "eta"})
        ws = smc.Workspace(dev)
        ref = _run(smc, "wait", mode, lp, lq, tok, ws, **kw)
        for variant in ("small", "poll256"):
            for rep in range(2):                 # twice on one workspace: the words were re-zeroed
                got = _run(smc, variant, mode, lp, lq, tok, ws, **kw)
                for f in ref:
                    assert torch.equal(_bits(ref[f]), _bits(got[f])), (variant, f, rep, ndv is not None)


@pytest.mark.parametrize("variant", ["small", "poll256", "wait"])
def test_tail_variant_staged_oracle_parity(smc, orc, variant):
    # the GPU's lam' (logw_pre) within 1e-4 of the oracle's, and the oracle's S4-S7 from it gives
    # the GPU's ancestry bit-exactly (reading G7: no ties here)
    P, N, K, V = 2, 16, 8, 128256
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=31, bonus=False)
    dev = torch.device("cuda")
    prev = synth.uniform_prior(P, N)
    _set(smc, variant)
    try:
        out = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), V=V, logw_prev=prev.to(dev),
                             eta=math.inf, seed=7, step=4, prompt_base=11)
        torch.cuda.synchronize()
    finally:
        _set(smc, "small")
    ref_w = orc.weights(to_host(lp), to_host(lq), tok.numpy(), V=V, logw_prev=prev.numpy())
    assert max_abs(np_(out.logw_pre), ref_w["logw"]) <= 1e-4
    staged = orc.resample(np_(out.logw_pre), eta=math.inf, seed=7, step=4, prompt_base=11)
    assert np.array_equal(np_(out.ancestors), staged["ancestors"])
    assert np.array_equal(np_(out.slot_src), staged["slot_src"])
    assert np.array_equal(np_(out.n_ties), staged["n_ties"])
    assert np.all(np_(out.status) == 0)


def test_small_tail_many_prompts(smc, orc):
    # thousands of one-CTA clusters (N K <= 16) queue behind the resident ones while K1 streams:
    # bit-identical to the wait tail, staged oracle parity on every prompt
    P, N, K, V = 3000, 2, 1, 100
    dev = torch.device("cuda")
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.float32, seed=77, bonus=False)
    lp, lq, tok = lp.to(dev), lq.to(dev), tok.to(dev)
    kw = dict(V=V, step=5, eta=math.inf)
    ws = smc.Workspace(dev)
    ref = _run(smc, "wait", "step", lp, lq, tok, ws, **kw)
    got = _run(smc, "small", "step", lp, lq, tok, ws, **kw)
    for f in ref:
        assert torch.equal(_bits(ref[f]), _bits(got[f])), f
    staged = orc.resample(np_(got["logw_pre"]), eta=math.inf, step=5)
    assert np.array_equal(np_(got["ancestors"]), staged["ancestors"])


@pytest.mark.parametrize("N,K,variant", [(16, 8, "small"), (64, 8, "small"), (12, 12, "small"),
                                         (16, 8, "poll256")])
def test_polling_tail_graph_replay_stress(smc, N, K, variant):
    """Back-to-back steps under CUDA-graph replay: a ring of 6 steps (each with its own inputs,
    step counter and outputs) captured once and replayed 150 times (900 steps, PDL-chained, the
    tail of one step overlapping the next step's K1 launch).  Each step's outputs after the last
    replay are bit-identical to the same step run eagerly: the work-counter gate, the word array
    zeroing and the counter re-arm carry no state from one step into the next."""
    dev = torch.device("cuda")
    V, R = 128256, 6
    ring = [synth.lm_logits(1, N, K, V, device=dev, seed=900 + 17 * r) for r in range(R)]
    _set(smc, variant)
    try:
        ws = smc.Workspace(dev)
        outs = [smc.Outputs() for _ in range(R)]
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())

        def steps():
            for i in range(R):
                smc.smcsd_step(*ring[i], V=V, eta=math.inf, step=i, out=outs[i], workspace=ws, stream=s)

        with torch.cuda.stream(s):
            steps()
        torch.cuda.synchronize()
        ref = [{f: getattr(o, f).clone() for f in FIELDS if getattr(o, f, None) is not None} for o in outs]
        for o in outs:                                          # poison: the replays must rewrite
            for f in ref[0]:
                getattr(o, f).fill_(7)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            steps()
        for _ in range(150):
            g.replay()
        torch.cuda.synchronize()
    finally:
        _set(smc, "small")
    for i, o in enumerate(outs):
        assert int(o.status.max()) == 0, i
        for f, t in ref[i].items():
            assert torch.equal(_bits(getattr(o, f)), _bits(t)), (i, f)
