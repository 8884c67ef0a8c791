#!/usr/bin/env python
"""Every libsmcsd entry point once on small shapes (cfg1 and a small cfg2), for
compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck}.  Usage (GPU):
  compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize.py"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc
import synth
from paper_2604_15672_b200.dist import TPExchange

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
for (P, N, K, V, dt) in ((1, 4, 4, 1000, torch.float32), (2, 16, 8, 20001, torch.bfloat16)):
    lp, lq, tok = (t.to(dev) for t in synth.lm_logits(P, N, K, V, dtype=dt, seed=5))
    ndr = torch.randint(0, K + 1, (P, N), dtype=torch.int32, device=dev)
    o = smc.smcsd_step(lp, lq, tok, V=V, n_drafted=ndr, step=1, bonus=True)
    smc.smcsd_step(lp, lq, tok, V=V, step=2, scheme=smc.SMCSD_MULTINOMIAL, eta=N / 2)   # polling tail
    smc.smcsd_set_poll_tail(False)                                   # wait-for-K1 tail
    smc.smcsd_step(lp, lq, tok, V=V, n_drafted=ndr, step=2, eta=N / 2)
    smc.smcsd_set_poll_tail(True)
    smc.smcsd_set_small_tail(False)                                  # 256-thread polling tail
    smc.smcsd_step(lp, lq, tok, V=V, n_drafted=ndr, step=2, eta=math.inf)
    smc.smcsd_weights(lp, lq, tok, V=V)
    smc.smcsd_set_small_tail(True)
    w = smc.smcsd_weights(lp, lq, tok, V=V, alpha=2.0)
    part = smc.smcsd_weights_partial(lp, lq, tok, v_begin=0, v_len=V)
    smc.smcsd_weights_combine(part.unsqueeze(0).contiguous(), tok, V=V)
    smc.smcsd_partials_rescale(part, part.clone())
    smc.smcsd_resample(w.logw, eta=math.inf, step=3)
    smc.smcsd_select(w.logw, step=4)
    smc.smcsd_powersmc_weights(lp[:, :, :1].contiguous(), V=V, alpha=2.5)
    smc.smcsd_powersmc_weights(lp[:, :, :1].contiguous(), V=V, alpha=3.0)
    smc.smcsd_powersmc_weights(lp[:, :, :1].contiguous(), V=V, alpha=0.5)      # half-integer path
    kv = synth.kv_bits((2, 2, P, N, 2, 64, 16), seed=1).to(dev)
    g = smc.kv_geometry(kv)
    dst = torch.empty_like(kv)
    smc.smcsd_kv_reindex(dst, kv, o.ancestors, **g)
    smc.smcsd_kv_reindex(kv, kv, o.slot_src, **g)
    hist = torch.randint(0, V, (P, N, 12), dtype=torch.int32, device=dev)
    smc.smcsd_kv_reindex_multi([smc.kv_tensor(kv, kv, **g),
                                smc.kv_tensor(hist, hist, n_outer=1, outer_stride=0, prompt_stride=N * 48,
                                              particle_stride=48, seg_count=1, seg_bytes=48, seg_stride=48)],
                               o.slot_src)
    PG = 4
    tab = torch.arange(P * N * PG, dtype=torch.int32, device=dev).view(P, N, PG)
    npg = torch.full((P, N), PG, dtype=torch.int32, device=dev)
    refc = torch.ones(P * N * PG, dtype=torch.int32, device=dev)
    smc.smcsd_kv_reindex_paged(tab, npg, refc, o.ancestors, freed=torch.zeros(P * N * PG, dtype=torch.uint8, device=dev))
    # paged append with copy-on-write of shared partial tails (after the paged resample above)
    refc_b = torch.ones(P * N * PG, dtype=torch.int32, device=dev)
    td, nd, _ = smc.smcsd_kv_reindex_paged(tab, npg, refc_b, o.ancestors)
    sl = torch.full((P, N), PG * 16 - 5, dtype=torch.int32, device=dev)
    rc2 = torch.cat([refc_b, torch.zeros(P * N * 2, dtype=torch.int32, device=dev)])
    pool = synth.kv_bits((2, rc2.numel(), 16, 2, 16), seed=3).to(dev)
    smc.smcsd_kv_append_paged(td, nd, sl, rc2, torch.full((P, N), 9, dtype=torch.int32, device=dev),
                              page_size=16, pools=(smc.kv_pool(pool, **smc.paged_pool_geometry(pool)),))
    # invalid reindex indices flag ST_BAD_INDEX (status output)
    bad = o.ancestors.clone()
    bad[:, 0] = N + 3
    st = torch.zeros(P, dtype=torch.int32, device=dev)
    smc.smcsd_kv_reindex(dst, kv, bad, status=st, **g)
    ex = TPExchange.local_group(P, N, K, V, 1, device=dev)[0]
    ex.step(lp, lq, tok, eta=math.inf, step=5)
    ex.close()
    torch.cuda.synchronize()
print("sanitize workload done", flush=True)
