"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (SURVEY.md
8(d)): the oracle checks sampled outputs it can compute one by one, and properties that hold at
any size check the rest.

* headline (configs[1]): bench.Cfg2Step itself -- smcsd_step (V=128256, N=16, K=8, bf16) + the
  in-place reindex of Llama-3.1-70B-shaped KV (80 x 2 x 8 x 2048 x 128 bf16, 640 MiB/particle)
  and of the token history.  Weights vs the oracle from the logits (1e-4), ancestors / slot
  plan vs the oracle's resampling of the GPU's fp32 log-weights (bit-exact), every KV block of
  every particle byte-equal to its source block (torch.equal against a copy taken before).
* configs[3]: 64 prompts x N=32 x K=8 in one launch; prompts 0, 37 and 63 against the oracle
  (Philox addressed by the global prompt index), every prompt against the invariants.
* configs[2]: 70B KV with N=32 (21.5 GB), pinned ancestor pattern, out of place and in place,
  every block checked.
"""
import argparse
import math
import os
import sys

import numpy as np
import pytest
import torch

import synth
from gpu_util import to_host

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL_LOGW = 1e-4


@pytest.fixture(scope="module")
def smc():
    import paper_2604_15672_b200 as m
    assert torch.cuda.is_available()
    return m


def _blocks_equal(kv_after, kv_before, src_index, p=0):
    """dst block n == src block src_index[n] for every (layer, K/V) plane: torch.equal on GPU."""
    idx = src_index.tolist()
    for n, a in enumerate(idx):
        if not torch.equal(kv_after[:, :, p, n], kv_before[:, :, p, a]):
            return n
    return -1


def test_headline_step_full_size(smc, orc):
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    import bench
    dev = torch.device("cuda")
    args = argparse.Namespace(warmup=1, steps=2, gpus=1)
    wl = bench.Cfg2Step(dev, 0, args)
    for i in range(3):
        lp, lq, tok = wl.ring[i % len(wl.ring)]
        prior = wl.logw.clone()
        kv0, hist0 = wl.kv.clone(), wl.hist.clone()
        wl.step(i)                                             # exactly the bench's launches
        torch.cuda.synchronize()
        assert int(wl.out.status[0]) == 0
        anc, slot = wl.anc[i, 0].cpu(), wl.slot[i, 0].cpu()
        # the KV and token reindex applied the slot plan, block by block
        assert _blocks_equal(wl.kv, kv0, slot) == -1
        assert torch.equal(wl.hist[0], hist0[0][slot.long()])
        del kv0, hist0
        # weights: a second call on the same inputs with logw_pre requested (same kernels)
        o2 = smc.smcsd_step(lp, lq, tok, V=wl.V, logw_prev=prior, eta=math.inf, seed=0x5EED5EED,
                            step=i, prompt_base=0)
        torch.cuda.synchronize()
        assert torch.equal(o2.ancestors[0].cpu(), anc) and torch.equal(o2.slot_src[0].cpu(), slot)
        ref_w = orc.weights(to_host(lp), to_host(lq), tok.cpu().numpy(), V=wl.V,
                            logw_prev=prior.cpu().numpy())
        gw = o2.logw_pre.cpu().numpy().astype(np.float64)
        assert np.max(np.abs(gw - ref_w["logw"])) <= TOL_LOGW
        ref_r = orc.resample(o2.logw_pre.cpu().numpy(), eta=math.inf, seed=0x5EED5EED, step=i)
        assert ref_r["n_ties"].sum() == 0
        assert np.array_equal(anc.numpy(), ref_r["ancestors"][0])
        assert np.array_equal(slot.numpy(), ref_r["slot_src"][0])
        assert abs(float(o2.ess[0]) - ref_r["ess"][0]) <= 1e-12 * ref_r["ess"][0]


def test_cfg4_full_size_sampled(smc, orc):
    dev = torch.device("cuda")
    P, N, K, V = 64, 32, 8, 128256
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, device=dev,
                                  seed=synth.GEN_SEED_BASE + 4)
    prior = synth.uniform_prior(P, N, device=dev)
    out = smc.smcsd_step(lp, lq, tok, V=V, logw_prev=prior, eta=math.inf, step=5, prompt_base=0)
    torch.cuda.synchronize()
    st = out.status.cpu().numpy()
    assert (st == 0).all()
    off = out.offspring.cpu().numpy()
    anc = out.ancestors.cpu().numpy()
    assert (off.sum(axis=1) == N).all() and (anc >= 0).all() and (anc < N).all()
    assert (np.diff(anc, axis=1) >= 0).all()                   # systematic: non-decreasing
    assert (out.logw.cpu().numpy() == orc.neg_log_n(N)).all()  # S7 reset everywhere
    for p in (0, 37, 63):
        ref_w = orc.weights(to_host(lp[p:p + 1]), to_host(lq[p:p + 1]), tok[p:p + 1].cpu().numpy(),
                            V=V, logw_prev=prior[p:p + 1].cpu().numpy())
        gw = out.logw_pre[p:p + 1].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(gw - ref_w["logw"])) <= TOL_LOGW, p
        ref_r = orc.resample(out.logw_pre[p:p + 1].cpu().numpy(), eta=math.inf, step=5, prompt_base=p)
        assert ref_r["n_ties"].sum() == 0
        assert np.array_equal(anc[p], ref_r["ancestors"][0]), p
        assert np.array_equal(out.slot_src[p].cpu().numpy(), ref_r["slot_src"][0]), p


@pytest.mark.parametrize("mode", ["out_of_place", "in_place"])
def test_cfg3_full_size(smc, orc, mode):
    dev = torch.device("cuda")
    N, L, H, S, d = 32, 80, 8, 2048, 128
    lw = torch.zeros((1, N), device=dev)
    lw[0, 1::2] = -float("inf")                                # 16 survivors x 2 offspring
    src = synth.kv_bits_fast((L, 2, 1, N, H, S, d), seed=7, device=dev)
    geom = smc.kv_geometry(src)
    o = smc.smcsd_resample(lw.clone(), eta=math.inf, step=2)
    torch.cuda.synchronize()
    ref = orc.resample(lw.cpu().numpy(), eta=math.inf, step=2)
    assert np.array_equal(o.ancestors.cpu().numpy(), ref["ancestors"])
    assert np.array_equal(o.slot_src.cpu().numpy(), ref["slot_src"])
    assert (o.offspring.cpu().numpy()[0, 0::2] == 2).all()
    before = src.clone()
    if mode == "out_of_place":
        dst = torch.empty_like(src)
        smc.smcsd_kv_reindex(dst, src, o.ancestors, **geom)
        torch.cuda.synchronize()
        assert _blocks_equal(dst, before, o.ancestors[0].cpu()) == -1
        assert torch.equal(src, before)                         # source untouched
    else:
        smc.smcsd_kv_reindex(src, src, o.slot_src, **geom)
        torch.cuda.synchronize()
        assert _blocks_equal(src, before, o.slot_src[0].cpu()) == -1
