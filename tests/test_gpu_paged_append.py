"""GPU parity of smcsd_kv_append_paged (paged append with copy-on-write, NEXT #1; PAPER.md:488-490,
SPEC.md:466-470, reading G24) against the oracle, bit for bit: tables, page counts, sequence
lengths, refcounts, slot mappings, the copy-on-write list, status / result and the KV pool bytes.
Multi-round: resample (smcsd_kv_reindex_paged) -> append, with the KV content of the new tokens
written through the slot mapping, on both sides; content is never copied by a resample."""
import numpy as np
import pytest
import torch

import synth
from gpu_util import np_

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def smc():
    import paper_2604_15672_b200 as m
    assert torch.cuda.is_available()
    return m


def _both(smc, orc, st, n_new, page, pool=None, max_new=None):
    """One append on the GPU (device copies of st) and in the oracle; returns both results."""
    dev = torch.device("cuda")
    table, npg, sl, rc = st
    d = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (table, npg, sl, rc)]
    nn = torch.from_numpy(np.ascontiguousarray(n_new, dtype=np.int32)).to(dev)
    pools, opools = (), ()
    if pool is not None:
        pd = torch.from_numpy(pool).to(dev)
        g = smc.paged_pool_geometry(pd)
        pools = (smc.kv_pool(pd, **g),)
        opools = ((pool.view(np.uint8).reshape(-1), g["n_planes"], g["plane_stride"], g["page_stride"],
                   g["token_bytes"]),)
    out = smc.smcsd_kv_append_paged(*d, nn, page_size=page, max_new=max_new, pools=pools)
    torch.cuda.synchronize()
    ref = orc.kv_append_paged(table, npg, sl, rc, n_new, page_size=page,
                              max_new=int(out.slot_mapping.shape[-1]), pools=opools)
    gpu = dict(table=np_(d[0]), n_pages=np_(d[1]), seq_len=np_(d[2]), refcount=np_(d[3]),
               slot_mapping=np_(out.slot_mapping), cow_src=np_(out.cow_src),
               cow_dst=np_(out.cow_dst), cow_tokens=np_(out.cow_tokens),
               status=np_(out.status).astype(np.uint32), result=int(np_(out.result)[0]))
    if pool is not None:
        gpu["pool"] = np_(pools[0][0])
    return gpu, ref


def _assert_same(gpu, ref, pool=None):
    assert gpu["result"] == ref["result"]
    assert np.array_equal(gpu["status"], ref["status"])
    for k in ("table", "n_pages", "seq_len", "refcount", "cow_src", "cow_dst", "cow_tokens"):
        assert np.array_equal(gpu[k], ref[k]), k
    if pool is not None and ref["result"] != 0:
        assert np.array_equal(gpu["pool"], pool)                 # an aborted call copies nothing
    if ref["result"] == 0:
        for k in ("slot_mapping", "cow_src", "cow_dst", "cow_tokens"):
            assert np.array_equal(gpu[k], ref[k]), k
        if pool is not None:
            assert np.array_equal(gpu["pool"], pool)


def _kv_pool(planes, num_pages, page, H, d, seed):
    return synth.kv_bits((planes, num_pages, page, H, d), seed=seed).numpy()


def test_spec_examples_and_shared_tails(smc, orc):
    P, N, MP, NUM, page = 2, 3, 6, 64, 16
    table = np.full((P, N, MP), -1, np.int32)
    npg = np.zeros((P, N), np.int32)
    sl = np.zeros((P, N), np.int32)
    rc = np.zeros(NUM, np.int32)
    # prompt 0: fresh particles (n = 16, 17, 0); prompt 1: three particles share a full page and a
    # 5-token tail (refcount 3), all append -> two copy-on-writes, the last keeps the tail
    table[1, :, 0] = 40
    table[1, :, 1] = 41
    npg[1] = 2
    sl[1] = page + 5
    rc[40] = rc[41] = 3
    pool = _kv_pool(4, NUM, page, 2, 16, seed=3)
    want_pool = pool.copy()
    gpu, ref = _both(smc, orc, (table, npg, sl, rc), [[16, 17, 0], [2, 2, 20]], page, pool=pool)
    orc.kv_append_paged(table, npg, sl, rc, np.array([[16, 17, 0], [2, 2, 20]], np.int32),
                        page_size=page, pools=((want_pool.view(np.uint8).reshape(-1), 4,
                                                NUM * page * 2 * 16 * 2, page * 2 * 16 * 2, 2 * 16 * 2),))
    _assert_same(gpu, ref, want_pool)
    assert ref["result"] == 0 and int((ref["cow_dst"][1] >= 0).sum()) == 2
    assert ref["table"][1, 2, 1] == 41 and ref["refcount"][41] == 1


@pytest.mark.parametrize("seed", range(6))
def test_random_rounds_bit_exact(smc, orc, seed):
    """Rounds of resample -> append with new-token KV written through the slot mapping, on the
    GPU and in the oracle from the same state each round; everything compared bit for bit."""
    rng = np.random.default_rng(seed)
    dev = torch.device("cuda")
    P, N, K, MP, page = int(rng.integers(1, 4)), int(rng.integers(2, 33)), 8, 24, 16
    NUM = P * N * MP
    H, d, planes = 2, 16, 3
    table = np.full((P, N, MP), -1, np.int32)
    npg = np.zeros((P, N), np.int32)
    sl = np.zeros((P, N), np.int32)
    rc = np.zeros(NUM, np.int32)
    pool = _kv_pool(planes, NUM, page, H, d, seed=100 + seed)
    # prompts of 21..60 tokens written by particle 0, then shared by every particle
    prompt = rng.integers(21, 61, size=P)
    n0 = np.zeros((P, N), np.int32)
    n0[:, 0] = prompt
    gpu, ref = _both(smc, orc, (table, npg, sl, rc), n0, page, pool=pool, max_new=64)
    _assert_same(gpu, ref, pool)
    st = (ref["table"], ref["n_pages"], ref["seq_len"], ref["refcount"])
    ident = np.zeros((P, N), np.int32)
    r = orc.kv_reindex_paged(st[0], st[1], st[3], ident)
    st = (r["table"], r["n_pages"], np.take_along_axis(st[2], ident, 1), r["refcount"])
    copies = 0
    for rnd in range(5):
        n_new = rng.integers(0, K + 2, size=(P, N)).astype(np.int32)
        if rnd == 0:
            n_new[:] = K + 1
        gpu, ref = _both(smc, orc, st, n_new, page, pool=pool.copy(), max_new=K + 1)
        want = pool.copy()
        orc.kv_append_paged(*st, n_new, page_size=page, max_new=K + 1,
                            pools=((want.view(np.uint8).reshape(-1), planes, NUM * page * H * d * 2,
                                    page * H * d * 2, H * d * 2),))
        _assert_same(gpu, ref, want)
        copies += int(ref["cow_tokens"].sum())
        # new tokens' KV (random bits) written at the slot mapping, the same on both sides
        pool = want
        sm = ref["slot_mapping"]
        flat = pool.reshape(planes, NUM * page, H * d)
        for s_ in sm[sm >= 0].tolist():
            flat[:, s_] = rng.integers(-30000, 30000, size=(planes, H * d), dtype=np.int16)
        st = (ref["table"], ref["n_pages"], ref["seq_len"], ref["refcount"])
        # resample on the GPU (paged reindex), checked against the oracle, no content moves
        lw = (rng.standard_normal((P, N)) * 1.5).astype(np.float32)
        a = orc.resample(lw, eta=np.inf, seed=rnd)["ancestors"]
        td, nd, stat = smc.smcsd_kv_reindex_paged(torch.from_numpy(st[0]).to(dev),
                                                  torch.from_numpy(st[1]).to(dev),
                                                  torch.from_numpy(st[3].copy()).to(dev),
                                                  torch.from_numpy(a).to(dev))
        torch.cuda.synchronize()
        r = orc.kv_reindex_paged(st[0], st[1], st[3], a)
        assert np.array_equal(np_(td), r["table"]) and np.array_equal(np_(nd), r["n_pages"])
        st = (r["table"], r["n_pages"], np.take_along_axis(st[2], a, 1), r["refcount"])
    assert copies > 0


def test_all_or_nothing(smc, orc):
    P, N, MP, NUM, page = 2, 2, 2, 3, 16
    base = (np.full((P, N, MP), -1, np.int32), np.zeros((P, N), np.int32), np.zeros((P, N), np.int32),
            np.zeros(NUM, np.int32))
    pool = _kv_pool(1, NUM, page, 1, 16, seed=2)
    gpu, ref = _both(smc, orc, base, [[16, 16], [16, 16]], page, pool=pool.copy())   # 4 pages > 3 free
    _assert_same(gpu, ref, pool)
    assert ref["result"] == 1 and ref["status"].tolist() == [128, 128]
    gpu, ref = _both(smc, orc, base, [[0, 48], [0, 0]], page)                # > max_pages
    _assert_same(gpu, ref)
    assert ref["result"] == 1 and ref["status"].tolist() == [16, 0]
    t, npg, sl, rc = (a.copy() for a in base)
    t[1, 0, 0] = 7                                                           # page id >= num_pages
    npg[1, 0] = 1
    sl[1, 0] = 3
    gpu, ref = _both(smc, orc, (t, npg, sl, rc), [[1, 0], [1, 0]], page)
    _assert_same(gpu, ref)
    assert ref["result"] == 1 and ref["status"].tolist() == [0, 16]
    # the workspace is left zeroed by an aborted call: a valid call right after is exact
    gpu, ref = _both(smc, orc, base, [[5, 16], [0, 1]], page)
    _assert_same(gpu, ref)
    assert ref["result"] == 0


def test_large_pool_lowest_free_ids(smc, orc):
    """A 70B-like page geometry (16-token pages, 8 KV heads x d 128 bf16 = 2 KiB per token) over
    many free-count chunks: allocation takes the lowest-id free pages, skipping used ones."""
    rng = np.random.default_rng(9)
    P, N, MP, page = 1, 32, 130, 16
    NUM = 12000
    rc = (rng.random(NUM) < 0.7).astype(np.int32)                          # 30% free, scattered
    table = np.full((P, N, MP), -1, np.int32)
    npg = np.zeros((P, N), np.int32)
    sl = np.zeros((P, N), np.int32)
    used = np.nonzero(rc)[0]
    for n in range(N):                                                      # each owns 2 pages + 3 tokens
        pages = used[3 * n:3 * n + 3]
        table[0, n, :3] = pages
        npg[0, n] = 3
        sl[0, n] = 2 * page + 3
    pool = _kv_pool(1, NUM, page, 8, 128, seed=5)
    gpu, ref = _both(smc, orc, (table, npg, sl, rc), np.full((P, N), 9, np.int32), page, pool=pool)
    want = pool.copy()
    orc.kv_append_paged(table, npg, sl, rc, np.full((P, N), 9, np.int32), page_size=page,
                        pools=((want.view(np.uint8).reshape(-1), 1, NUM * page * 8 * 128 * 2,
                                page * 8 * 128 * 2, 8 * 128 * 2),))
    _assert_same(gpu, ref, want)
    assert (ref["cow_dst"] == -1).all()                                     # exclusive tails
