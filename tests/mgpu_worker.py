"""Worker for tests/test_gpu_multigpu.py (launched by torchrun, one process per GPU; not a test
module itself).  On the ranks' own devices it checks the two sharded axes of SURVEY.md 8(e):

  DP  every rank runs smcsd_step on its prompt shard (global prompt index for Philox); rank 0
      gathers the shards and compares them BIT FOR BIT with a single-device run of all prompts;
  TP  the fused peer-memory step (smcsd_tp_step over CUDA-IPC-mapped buffers on the other GPUs)
      must give bit-identical weights / ancestors on every rank, within 1e-4 of the oracle's
      weights and with the oracle's ancestors from the staged fp32 log-weights; and, when every
      rank has its own GPU, the NCCL all-gather form (tp_weights over a nccl group) agrees.

Prints "rank R OK" or "rank R FAIL ..." and exits non-zero on failure."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_15672_b200 as smc  # noqa: E402
import synth  # noqa: E402
from paper_2604_15672_b200.dist import TPExchange, prompt_shard, tp_weights  # noqa: E402


def gather_to_all(t):
    """all_gather of a CPU tensor (gloo plumbing)."""
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t.contiguous())
    return out


def check_dp(rank, world, dev, fails):
    P, N, K, V = 2 * world, 16, 4, 30000
    lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=501)   # same everywhere
    b, e = prompt_shard(P, world, rank)
    kw = dict(V=V, eta=math.inf, seed=99, step=3)
    part = smc.smcsd_step(lp[b:e].contiguous().to(dev), lq[b:e].contiguous().to(dev),
                          tok[b:e].contiguous().to(dev), prompt_base=b, **kw)
    torch.cuda.synchronize(dev)
    mine = torch.cat([part.logw_pre.cpu().view(torch.int32).flatten(), part.ancestors.cpu().flatten(),
                      part.slot_src.cpu().flatten(), part.logw.cpu().view(torch.int32).flatten()])
    allp = gather_to_all(mine)
    if rank == 0:
        full = smc.smcsd_step(lp.to(dev), lq.to(dev), tok.to(dev), prompt_base=0, **kw)
        torch.cuda.synchronize(dev)
        for g in range(world):
            gb, ge = prompt_shard(P, world, g)
            sl = slice(gb, ge)
            want = torch.cat([full.logw_pre[sl].cpu().view(torch.int32).flatten(),
                              full.ancestors[sl].cpu().flatten(), full.slot_src[sl].cpu().flatten(),
                              full.logw[sl].cpu().view(torch.int32).flatten()])
            if not torch.equal(allp[g], want):
                fails.append(f"DP shard of rank {g} differs from the single-device run")


def check_tp(rank, world, dev, fails):
    import oracle
    P, N, K, V = 1, 16, 4, 50000
    ex = TPExchange(P, N, K, V)
    ws = smc.Workspace(dev)
    for it in range(3):
        lp, lq, tok = synth.lm_logits(P, N, K, V, dtype=torch.bfloat16, seed=77 + it)
        b, e = ex.v_begin, ex.v_begin + ex.v_len
        w = (e - b + 7) // 8 * 8
        sp = torch.zeros((P, N, K + 1, w), dtype=torch.bfloat16)
        sq = torch.zeros((P, N, K, w), dtype=torch.bfloat16)
        sp[..., :e - b] = lp[..., b:e]
        sq[..., :e - b] = lq[..., b:e]
        out = ex.step(sp.to(dev), sq.to(dev), tok.to(dev), eta=math.inf, seed=5, step=it, workspace=ws)
        torch.cuda.synchronize(dev)
        if int(out.status.max().item()) != 0:
            fails.append(f"TP step {it}: status {out.status.tolist()}")
        mine = torch.cat([out.logw_pre.cpu().view(torch.int32).flatten(), out.ancestors.cpu().flatten()])
        allv = gather_to_all(mine)
        if not all(torch.equal(allv[0], a) for a in allv):
            fails.append(f"TP step {it}: ranks disagree")
        if rank == 0:
            u16 = lambda t: t.view(torch.int16).numpy().view(np.uint16)
            ref = oracle.weights(u16(lp), u16(lq), tok.numpy(), V=V)
            err = float(np.max(np.abs(out.logw_pre.cpu().numpy().astype(np.float64) - ref["logw"])))
            if err > 1e-4:
                fails.append(f"TP step {it}: |logw - oracle| = {err:.2e}")
            st = oracle.resample(out.logw_pre.cpu().numpy(), eta=math.inf, seed=5, step=it)
            ok = st["n_ties"] == 0
            if not np.array_equal(out.ancestors.cpu().numpy()[ok], st["ancestors"][ok]):
                fails.append(f"TP step {it}: ancestors differ from the oracle's staged resample")
        # the NCCL all-gather form, when every rank has its own device
        if torch.cuda.device_count() >= world and world > 1:
            if not hasattr(check_tp, "nccl"):
                check_tp.nccl = dist.new_group(backend="nccl")
            wo = tp_weights(sp.to(dev), sq.to(dev), tok.to(dev), V=V, v_begin=b, v_len=e - b,
                            group=check_tp.nccl)
            torch.cuda.synchronize(dev)
            d = float((wo.logw - out.logw_pre).abs().max().item())
            if d > 1e-5:
                fails.append(f"TP step {it}: NCCL all-gather form differs from the fused step by {d:.2e}")
    ex.close()


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    fails = []
    check_dp(rank, world, dev, fails)
    check_tp(rank, world, dev, fails)
    dist.barrier()
    print(f"rank {rank} {'OK' if not fails else 'FAIL ' + '; '.join(fails)} (device {dev}, world {world})",
          flush=True)
    dist.destroy_process_group()
    sys.exit(0 if not fails else 1)


if __name__ == "__main__":
    main()
