"""Multi-GPU host logic (one process per GPU, torch.distributed for the plumbing).

The path shards along the two axes SURVEY.md 8(e) names:
  * prompts (data parallel): rank g owns prompts [g*P/G, (g+1)*P/G); no data-path collective;
    the Philox stream is addressed by the GLOBAL prompt index (prompt_base), so every rank's
    results equal a single-GPU run bit for bit.
  * vocabulary (tensor parallel, cfg5): rank g owns columns [b_g, b_{g+1}) of every logit row;
    smcsd_weights_partial -> all_gather of 16 B per row (S10) -> smcsd_weights_combine, which
    merges shards in rank order so every rank obtains bit-identical weights and ancestors.
This module holds the partitioning and the exchange only; all arithmetic is in libsmcsd.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def prompt_shard(P: int, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of the prompts owned by `rank` (contiguous, balanced to within one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(P, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def vocab_shard(V: int, world: int, rank: int, align: int = 8) -> tuple[int, int]:
    """[begin, end) of the vocabulary columns owned by `rank`.  Boundaries are multiples of
    `align` columns (16-byte rows for bf16) except the final end = V."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    units = (V + align - 1) // align
    base, extra = divmod(units, world)
    b = (rank * base + min(rank, extra)) * align
    e = b + (base + (1 if rank < extra else 0)) * align
    return min(b, V), min(e, V)


def exchange_partials(partials: torch.Tensor, group=None) -> torch.Tensor:
    """S10: gather every rank's [P][2][N][K][4] partials into [G][...] in rank order."""
    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(partials.shape), dtype=partials.dtype,
                      device=partials.device)
    exchange_partials_into(out, partials, group)
    return out


def exchange_partials_into(out: torch.Tensor, partials: torch.Tensor, group=None) -> None:
    """S10 into a preallocated [G][...] buffer (NCCL all_gather_into_tensor over NVLink; gloo
    stages through host memory -- functional tests only)."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, partials.contiguous(), group=group)
        return
    host = partials.detach().cpu().contiguous()
    bufs = [torch.empty_like(host) for _ in range(dist.get_world_size(group))]
    dist.all_gather(bufs, host, group=group)
    out.copy_(torch.stack(bufs))


def max_over_ranks(value: float, device, group=None) -> float:
    """Max of a host float over ranks (timing: the slowest rank sets the step time)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    if dist.get_backend(group) == "gloo":
        device = "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def tp_weights(logits_p_shard, logits_q_shard, tokens, *, V, v_begin, v_len, group=None, **kw):
    """Tensor-parallel S1-S4: partial on this rank's shard, gather, combine (rank order)."""
    import paper_2604_15672_b200 as smc
    part = smc.smcsd_weights_partial(logits_p_shard, logits_q_shard, tokens, v_begin=v_begin,
                                     v_len=v_len, n_drafted=kw.get("n_drafted"),
                                     inv_temp_p=kw.get("inv_temp_p", 1.0),
                                     inv_temp_q=kw.get("inv_temp_q", 1.0),
                                     workspace=kw.get("workspace"))
    gathered = exchange_partials(part, group)
    return smc.smcsd_weights_combine(gathered, tokens, V=V, n_drafted=kw.get("n_drafted"),
                                     logw_prev=kw.get("logw_prev"), alpha=kw.get("alpha", 1.0),
                                     out=kw.get("out"), workspace=kw.get("workspace_combine"))
