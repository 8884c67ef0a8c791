"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in paper_2604_15672_b200/dist.py:
prompt sharding with global Philox addressing (DP) and the vocab-shard exchange (TP).  The
per-shard arithmetic here is the oracle's; on the GPU the same host logic drives libsmcsd."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_15672_b200.dist import exchange_partials, max_over_ranks, prompt_shard, vocab_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    return res


def test_shard_ranges():
    for P in (1, 5, 64):
        for G in (1, 2, 3, 8):
            spans = [prompt_shard(P, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == P
            assert all(spans[i][1] == spans[i + 1][0] for i in range(G - 1))
    for V in (1000, 128256, 8193):
        for G in (1, 2, 4, 8):
            spans = [vocab_shard(V, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == V
            assert all(s[0] % 8 == 0 for s in spans)
            assert all(spans[i][1] == spans[i + 1][0] for i in range(G - 1))
    assert vocab_shard(128256, 8, 3) == (48096, 64128)


def _dp_job(rank, world):
    import oracle
    oracle.build()
    rng = np.random.default_rng(5)
    lw = (rng.standard_normal((6, 24)) * 2).astype(np.float32)
    b, e = prompt_shard(6, world, rank)
    mine = oracle.resample(lw[b:e], eta=np.inf, seed=77, step=3, prompt_base=b)
    t = torch.from_numpy(mine["ancestors"].copy())
    sizes = [prompt_shard(6, world, g)[1] - prompt_shard(6, world, g)[0] for g in range(world)]
    bufs = [torch.zeros((s, 24), dtype=torch.int32) for s in sizes]
    dist.all_gather(bufs, t)
    full = oracle.resample(lw, eta=np.inf, seed=77, step=3)
    slow = max_over_ranks(float(rank + 1), "cpu")
    return bool(np.array_equal(torch.cat(bufs).numpy(), full["ancestors"])) and slow == world


def test_dp_prompt_sharding_gloo():
    res = _run(_dp_job)
    assert res == {0: True, 1: True}


def _tp_job(rank, world):
    import oracle
    oracle.build()
    rng = np.random.default_rng(9)
    V, rows = 1000, 6
    z = (rng.standard_normal((rows, V)) * 3).astype(np.float32)
    d = rng.integers(0, V, rows)
    b, e = vocab_shard(V, world, rank)
    part = np.stack([oracle.row_partial(z[r, b:e], b, int(d[r]))[0] for r in range(rows)])
    gathered = exchange_partials(torch.from_numpy(part)).numpy()        # [G][rows][3]
    ok = True
    for r in range(rows):
        ell, flag = oracle.combine_partials(gathered[:, r, :])
        ref, _ = oracle.row_logprob(z[r], int(d[r]))
        ok &= flag == 0 and abs(ell - ref) <= 1e-12
    return bool(ok), gathered.tobytes()


def test_tp_vocab_exchange_gloo():
    res = _run(_tp_job)
    assert res[0][0] and res[1][0]
    assert res[0][1] == res[1][1]            # every rank holds the same gathered bytes


def _tp_allreduce_job(rank, world):
    # S10 all-reduce form (north star: "all-reduces the per-row max/sum-exp"): MAX of {m, x},
    # rescale to the global max (a CPU reference of smcsd_partials_rescale, natural-log units as
    # the oracle's partials), SUM of s; the merged row gives the unsharded log-prob
    import oracle
    from paper_2604_15672_b200.dist import exchange_partials_allreduce
    oracle.build()
    rng = np.random.default_rng(9)
    V, rows = 1000, 6
    z = (rng.standard_normal((rows, V)) * 3).astype(np.float32)
    d = rng.integers(0, V, rows)
    b, e = vocab_shard(V, world, rank)
    p3 = np.stack([oracle.row_partial(z[r, b:e], b, int(d[r]))[0] for r in range(rows)])
    part = torch.from_numpy(np.concatenate([p3, np.zeros((rows, 1))], axis=1))   # {m, s, x, 0}

    def rescale_ref(local, mx):
        out = mx.clone()
        s = local[:, 1] * torch.exp(local[:, 0] - mx[:, 0])
        out[:, 1] = torch.where(local[:, 1] == 0, torch.zeros_like(s), s)
        out[:, 3] = 0
        return out
    merged = exchange_partials_allreduce(part, rescale=rescale_ref).numpy()       # [1][rows][4]
    ok = True
    for r in range(rows):
        ell, flag = oracle.combine_partials(merged[:, r, :3])
        ref, _ = oracle.row_logprob(z[r], int(d[r]))
        ok &= flag == 0 and abs(ell - ref) <= 1e-12
    return bool(ok), merged.tobytes()


def test_tp_vocab_allreduce_gloo():
    res = _run(_tp_allreduce_job)
    assert res[0][0] and res[1][0]
    assert res[0][1] == res[1][1]            # every rank holds the same merged rows


def _handles_fn(rank, world):
    # S10 fused path plumbing: every rank's (fake) IPC handle reaches every rank in rank order,
    # and the peer table keeps our own buffer and opens only the peers'
    from paper_2604_15672_b200.dist import peer_table, share_handles
    h = bytes([rank]) * 64
    hs = share_handles(h)
    opened = []
    tab = peer_table(hs, rank, 1000 + rank, lambda b: opened.append(b[0]) or 5000 + b[0])
    return hs, tab, opened


def test_tp_exchange_handle_plumbing_gloo():
    res = _run(_handles_fn)
    for r in (0, 1):
        hs, tab, opened = res[r]
        assert hs == [bytes([0]) * 64, bytes([1]) * 64]
        assert tab[r] == 1000 + r and tab[1 - r] == 5000 + (1 - r)
        assert opened == [1 - r]


def _open_peers_fn(rank, world, fail_rank):
    # open_peers: a failure to open a peer on one rank raises on EVERY rank (no rank is left in
    # a later collective), and the peers a rank did open are closed again
    from paper_2604_15672_b200.dist import open_peers, share_handles
    hs = share_handles(bytes([rank]) * 8)
    closed = []

    def open_fn(b):
        if rank == fail_rank:
            raise OSError("no peer access")
        return 5000 + b[0]

    try:
        tab = open_peers(hs, rank, 1000 + rank, open_fn, lambda p, h: closed.append(p))
        return ("ok", tab, closed)
    except RuntimeError as e:
        return ("raised", str(e), closed)


def _open_ok(rank, world):
    return _open_peers_fn(rank, world, fail_rank=-1)


def _open_fail(rank, world):
    return _open_peers_fn(rank, world, fail_rank=1)


def test_open_peers_agreement_gloo():
    res = _run(_open_ok)
    assert res[0] == ("ok", [1000, 5001], []) and res[1] == ("ok", [5000, 1001], [])
    res = _run(_open_fail)
    assert res[0][0] == "raised" and res[1][0] == "raised"
    assert res[0][2] == [5001]                  # rank 0 opened rank 1's buffer, then closed it
    assert "no peer access" in res[1][1]


def test_xnseg_covers_every_shard():
    from paper_2604_15672_b200.dist import xnseg_for
    assert xnseg_for(128256, 8) == 2 and xnseg_for(128256, 1) == 16 and xnseg_for(128256, 4) == 4
    for V in (1000, 8193, 50001):
        for G in (1, 2, 3, 8):
            w = max(e - b for b, e in (vocab_shard(V, G, g) for g in range(G)))
            assert xnseg_for(V, G) * 8192 >= w > (xnseg_for(V, G) - 1) * 8192
