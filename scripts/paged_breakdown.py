#!/usr/bin/env python
"""Per-call device time of one paged engine round at the 70B shape (bench.measure_paged_round's
inputs): resample, paged reindex, seq_len gather, paged append.  Usage (GPU)."""
import math, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_15672_b200 as smc

dev = torch.device("cuda")
N, page, K1 = 32, 16, 9
L, H, S, d = 80, 8, 2048, 128
seq0 = S - K1 - 3
PG = (S + page - 1) // page + 1
own = (seq0 + page - 1) // page
num_pages = N * own + N * 2 + 64
planes = int(os.environ.get("PLANES", L * 2))
pool = torch.empty((planes, num_pages, page, H, d), dtype=torch.bfloat16, device=dev)
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
o, ao = smc.Outputs(), smc.AppendOutputs()
pools = (smc.kv_pool(pool, **geom),)
names = ["resample", "reindex_paged", "seq_len gather", "append_paged"]
acc = {k: [] for k in names}
for it in range(12):
    tab.copy_(tab0); npg.copy_(npg0); sl.copy_(sl0); rc.copy_(rc0)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    r = smc.smcsd_resample(lw, eta=math.inf, step=it, out=o)
    ev[1].record()
    smc.smcsd_kv_reindex_paged(tab, npg, rc, r.ancestors, table_dst=tab2, n_pages_dst=npg2)
    ev[2].record()
    sl.copy_(torch.gather(sl, 1, r.ancestors.long()))
    ev[3].record()
    smc.smcsd_kv_append_paged(tab2, npg2, sl, rc, nn, page_size=page, max_new=K1, pools=pools, out=ao)
    ev[4].record()
    torch.cuda.synchronize()
    if it >= 2:
        for j, k in enumerate(names):
            acc[k].append(ev[j].elapsed_time(ev[j + 1]) * 1e3)
print("planes", planes, " ".join(f"{k}: {statistics.median(v):.1f} us" for k, v in acc.items()),
      "result", int(ao.result.item()), "cow", int((ao.cow_dst >= 0).sum().item()))
