#!/usr/bin/env python
"""Two (or more) processes, one GPU each (or all on cuda:0 of a 1-GPU box), CUDA IPC: the fused
TP step (smcsd_tp_step) with a real cross-process exchange (IPC-mapped peer buffers).  Checks every rank gets
bit-identical results and that they match the single-process smcsd_step within 1e-4.
Launch: torchrun --nproc-per-node 2 scripts/tp_multiproc.py   (gloo for the plumbing)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2604_15672_b200 as smc
import synth
from paper_2604_15672_b200.dist import TPExchange


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    # one device per rank when the box has them (real NVLink P2P between ranks); on a 1-GPU box
    # every rank shares cuda:0 (time-sliced contexts, the IPC path still crosses processes)
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    P, N, K, V = 1, 16, 4, 50000
    pad = torch.empty(12345 + 777 * rank, dtype=torch.uint8, device=dev)  # buffer at an offset
    ex = TPExchange(P, N, K, V)
    ws = smc.Workspace(dev)
    ok = True
    for it in range(3):
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, device=dev, seed=77 + it)
        b, e = ex.v_begin, ex.v_begin + ex.v_len
        w = (e - b + 7) // 8 * 8
        sp = torch.zeros((P, N, K + 1, w), dtype=torch.bfloat16, device=dev)
        sq = torch.zeros((P, N, K, w), dtype=torch.bfloat16, device=dev)
        sp[..., :e - b] = lp[..., b:e]
        sq[..., :e - b] = lq[..., b:e]
        out = ex.step(sp, sq, tok, eta=math.inf, step=it, workspace=ws)
        torch.cuda.synchronize()
        full = smc.smcsd_step(lp, lq, tok, V=V, eta=math.inf, step=it)
        torch.cuda.synchronize()
        mine = torch.cat([out.logw_pre.flatten().cpu(), out.ancestors.flatten().float().cpu()])
        allv = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allv, mine)
        same = all(torch.equal(allv[0], a) for a in allv)
        err = (out.logw_pre - full.logw_pre).abs().max().item()
        st = int(out.status.max().item())
        ok &= same and err <= 1e-4 and st == 0
        print(f"rank {rank} step {it}: identical across ranks {same}, |logw - unsharded| {err:.2e}, "
              f"status {st}, ancestors equal to unsharded {torch.equal(out.ancestors, full.ancestors)}",
              flush=True)
    ex.close()
    dist.barrier()
    dist.destroy_process_group()
    print(f"rank {rank} {'OK' if ok else 'FAIL'}", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
