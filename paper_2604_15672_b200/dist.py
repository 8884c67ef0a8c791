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


def _all_reduce(t: torch.Tensor, op, group=None) -> None:
    """In-place all-reduce (NCCL on device; gloo stages through host memory -- tests only)."""
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=op, group=group)
        return
    host = t.detach().cpu().contiguous()
    dist.all_reduce(host, op=op, group=group)
    t.copy_(host)


def exchange_partials_allreduce(partials: torch.Tensor, group=None, rescale=None) -> torch.Tensor:
    """S10 in the north star's all-reduce form (include/smcsd.h, smcsd_partials_rescale):
    all_reduce(MAX) of the partials {m, s, x, 0} (m and x used), this rank's sums rescaled to
    the global max by our kernel, all_reduce(SUM) of the rescaled sums.  Returns [1][...][4]
    merged rows {M, S, X, 0} for smcsd_weights_combine with G = 1 -- identical on every rank,
    but S summed in NCCL's order (the all-gather path merges in rank order instead).
    rescale: the step-3 function (default: the CUDA kernel; CPU tests pass a reference)."""
    if rescale is None:
        import paper_2604_15672_b200 as smc
        rescale = smc.smcsd_partials_rescale
    mx = partials.clone()
    _all_reduce(mx, dist.ReduceOp.MAX, group)
    out = rescale(partials, mx)
    s = out[..., 1].contiguous()
    _all_reduce(s, dist.ReduceOp.SUM, group)
    out[..., 1] = s
    return out.unsqueeze(0)


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
    """Tensor-parallel S1-S4: partial on this rank's shard, exchange (exchange="allgather":
    rank-order merge, bit-identical to one GPU; "allreduce": MAX + rescale + SUM), combine."""
    import paper_2604_15672_b200 as smc
    part = smc.smcsd_weights_partial(logits_p_shard, logits_q_shard, tokens, v_begin=v_begin,
                                     v_len=v_len, n_drafted=kw.get("n_drafted"),
                                     inv_temp_p=kw.get("inv_temp_p", 1.0),
                                     inv_temp_q=kw.get("inv_temp_q", 1.0),
                                     workspace=kw.get("workspace"))
    gathered = (exchange_partials_allreduce(part, group) if kw.get("exchange") == "allreduce"
                else exchange_partials(part, group))
    return smc.smcsd_weights_combine(gathered, tokens, V=V, n_drafted=kw.get("n_drafted"),
                                     logw_prev=kw.get("logw_prev"), alpha=kw.get("alpha", 1.0),
                                     out=kw.get("out"), workspace=kw.get("workspace_combine"))


# ------------------------------------------------------------------------------------------
# S10 fused into K1 over peer memory (smcsd_tp_step): the exchange buffers.
# ------------------------------------------------------------------------------------------
def share_handles(handle: bytes, group=None) -> list[bytes]:
    """All ranks' IPC handles in rank order (plumbing over torch.distributed, any backend)."""
    world = dist.get_world_size(group)
    got: list = [None] * world
    dist.all_gather_object(got, handle, group=group)
    return [bytes(h) for h in got]


def peer_table(handles: list[bytes], rank: int, local_ptr: int, open_fn) -> list[int]:
    """Device addresses of every rank's exchange buffer as seen by this process: our own
    buffer directly, every peer's through open_fn(handle) (cudaIpcOpenMemHandle)."""
    return [local_ptr if g == rank else int(open_fn(h)) for g, h in enumerate(handles)]


def open_peers(handles: list[bytes], rank: int, local_ptr: int, open_fn, close_fn, group=None,
               device="cpu") -> list[int]:
    """peer_table with an all-rank agreement: every rank reaches the all-reduce even when
    opening a peer fails on it, so a failure raises on every rank (and the peers it did open
    are closed) instead of leaving the other ranks blocked in a later collective."""
    err, ptrs = None, None
    try:
        ptrs = peer_table(handles, rank, local_ptr, open_fn)
    except Exception as exc:  # depends on the machine's P2P / IPC support
        err = exc
    bad = torch.tensor([0.0 if err is None else 1.0],
                       device=device if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=group)
    if float(bad.item()) != 0.0:
        if ptrs is not None:
            for g, p in enumerate(ptrs):
                if g != rank:
                    close_fn(p, handles[g])
        raise RuntimeError(f"opening the peers' exchange buffers failed on some rank "
                           f"(this rank: {err!r})")
    return ptrs


def xnseg_for(V: int, world: int, align: int = 8) -> int:
    """Segment slots per rank: the widest shard's ceil(width / SMCSD_SEGMENT), same on all ranks."""
    seg = 8192
    return max((e - b + seg - 1) // seg for b, e in (vocab_shard(V, world, g, align) for g in range(world)))


class TPExchange:
    """One rank's exchange buffer plus the peer address table for smcsd_tp_step.

    Multi-process: TPExchange(P, N, K, V, group=...) exports this rank's buffer, gathers every
    rank's handle (torch.distributed) and opens the peers' buffers (CUDA IPC, NVLink P2P).
    Single process: TPExchange.local_group(...) returns G exchanges whose tables point at each
    other's buffers on one device (G simulated ranks; run each on its own stream)."""

    def __init__(self, P, N, K, V, *, group=None, device=None, world=None, rank=None, _buf=None,
                 device_epoch=True):
        import paper_2604_15672_b200 as smc
        self.smc = smc
        self.device = torch.device("cuda" if device is None else device)
        self.G = dist.get_world_size(group) if world is None else world
        self.rank = dist.get_rank(group) if rank is None else rank
        self.P, self.N, self.K, self.V = P, N, K, V
        self.xnseg = xnseg_for(V, self.G)
        self.v_begin, v_end = vocab_shard(V, self.G, self.rank)
        self.v_len = v_end - self.v_begin
        self.nbytes = smc.smcsd_tp_exchange_bytes(P, N, K, self.G, self.xnseg)
        self.buf = _buf if _buf is not None else torch.empty(self.nbytes, dtype=torch.uint8, device=self.device)
        smc.smcsd_tp_exchange_init(self.buf)
        self.epoch = 0
        # device_epoch: the epoch lives in the exchange buffer and advances on the GPU, so a
        # step captured in a CUDA graph stays correct on replay; False: host epoch per call
        self.device_epoch = device_epoch
        self._opened: list[int] = []
        self.xpeer = None
        # this rank's own workspace: simulated ranks run concurrently on separate streams and
        # must not share counters / partials (include/smcsd.h: no sharing by concurrent calls)
        self.ws = smc.Workspace(self.device)
        if world is None:                      # multi-process: share handles, open peers
            torch.cuda.synchronize(self.device)
            handles = share_handles(smc.smcsd_ipc_export(self.buf), group)
            ptrs = open_peers(handles, self.rank, self.buf.data_ptr(), smc.smcsd_ipc_open,
                              smc.smcsd_ipc_close, group=group, device=self.device)
            self._opened = [(p, handles[g]) for g, p in enumerate(ptrs) if g != self.rank]
            self.set_peers(ptrs)
            dist.barrier(group)                # every buffer initialised before any push

    def set_peers(self, ptrs: list[int]):
        self.xpeer = torch.tensor(ptrs, dtype=torch.int64, device=self.device)

    @classmethod
    def local_group(cls, P, N, K, V, G, device=None, device_epoch=True):
        ex = [cls(P, N, K, V, device=device, world=G, rank=g, device_epoch=device_epoch) for g in range(G)]
        ptrs = [e.buf.data_ptr() for e in ex]
        for e in ex:
            e.set_peers(ptrs)
        torch.cuda.synchronize(ex[0].device)
        return ex

    def step(self, logits_p_shard, logits_q_shard, tokens, **kw):
        """One smcsd_tp_step: device-resident epoch (graph-capturable), or the host epoch
        advanced here (identical on every rank)."""
        self.epoch += 1
        kw.setdefault("workspace", self.ws)
        return self.smc.smcsd_tp_step(logits_p_shard, logits_q_shard, tokens, V=self.V,
                                      v_begin=self.v_begin, v_len=self.v_len, rank=self.rank,
                                      G=self.G, xnseg=self.xnseg,
                                      epoch=0 if self.device_epoch else self.epoch,
                                      xpeer=self.xpeer, xlocal=self.buf, **kw)

    def close(self):
        for p, h in self._opened:
            self.smc.smcsd_ipc_close(p, h)
        self._opened = []
