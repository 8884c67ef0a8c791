"""Pins for the paged append / copy-on-write oracle (NEXT #1; Sec. 3.3 Obs. 2;
SPEC.md:466-470 append_tokens, reading G24).

Pinned against SPEC's worked examples, refcount conservation, and a brute-force
model: a plain list of tokens per particle.  Resample (orc.kv_reindex_paged) + append with the
new tokens written through slot_mapping must leave every particle's page list spelling out
exactly its ancestor's tokens followed by its own new ones, and no call may write into a page
another particle can see (the property copy-on-write exists for)."""
import numpy as np
import pytest

PAGE = 16


def _state(P, N, MP, num_pages):
    return (np.full((P, N, MP), -1, np.int32), np.zeros((P, N), np.int32),
            np.zeros((P, N), np.int32), np.zeros(num_pages, np.int32))


def _append(orc, st, n_new, pool=None, **kw):
    table, npg, sl, rc = st
    pools = [] if pool is None else [(pool, 1, 0, PAGE * 4, 4)]     # one plane, int32 tokens
    out = orc.kv_append_paged(table, npg, sl, rc, np.asarray(n_new, np.int32), page_size=PAGE,
                              pools=pools, **kw)
    return out, (out["table"], out["n_pages"], out["seq_len"], out["refcount"])


def test_spec_examples_fresh_pages(orc):
    # fresh particle, n = capacity -> exactly 1 page; n = capacity + 1 -> 2 pages,
    # the second with 1 token
    st = _state(1, 2, 4, 8)
    out, st = _append(orc, st, [[PAGE, PAGE + 1]])
    assert out["result"] == 0
    assert out["n_pages"].tolist() == [[1, 2]] and out["seq_len"].tolist() == [[16, 17]]
    assert out["table"][0, 0, :1].tolist() == [0] and out["table"][0, 1, :2].tolist() == [1, 2]
    assert out["refcount"].tolist() == [1, 1, 1, 0, 0, 0, 0, 0]
    assert out["slot_mapping"][0, 1, 16] == 2 * PAGE + 0                # token 17: page 2 slot 0
    assert (out["cow_dst"] == -1).all()


def test_full_shared_page_is_never_copied(orc):
    # two particles share a full prefix page; one appends -> a fresh page, no copy
    table, npg, sl, rc = _state(1, 2, 4, 8)
    table[0, :, 0] = 5
    npg[:] = 1
    sl[:] = PAGE
    rc[5] = 2
    out, _ = _append(orc, (table, npg, sl, rc), [[3, 0]])
    assert out["result"] == 0 and (out["cow_dst"] == -1).all() and out["cow_tokens"].sum() == 0
    assert out["table"][0, 0, :2].tolist() == [5, 0] and out["refcount"][5] == 2
    assert out["slot_mapping"][0, 0, :3].tolist() == [0, 1, 2]


@pytest.mark.parametrize("appenders,copies", [((1, 0, 0), 1), ((1, 1, 0), 2), ((1, 1, 1), 2),
                                              ((0, 1, 1), 2), ((0, 0, 1), 1)])
def test_shared_partial_tail_copy_on_write(orc, appenders, copies):
    """Three particles share a tail page holding 5 tokens (refcount 3).  In (p, n) order each
    appender sees the current refcount: > 1 -> copy-on-write (copies the 5 filled tokens, not the
    page), = 1 -> fills in place.  So with all three appending the first two copy and the last
    keeps the page; with fewer appenders every appender copies."""
    table, npg, sl, rc = _state(1, 3, 4, 16)
    table[0, :, 0] = 7
    table[0, :, 1] = 9
    npg[:] = 2
    sl[:] = PAGE + 5
    rc[7] = rc[9] = 3
    pool = np.full(16 * PAGE, -1, np.int32)
    pool[7 * PAGE:8 * PAGE] = np.arange(100, 116)
    pool[9 * PAGE:9 * PAGE + 5] = np.arange(200, 205)
    out, _ = _append(orc, (table, npg, sl, rc), [list(appenders)], pool=pool.view(np.uint8))
    assert out["result"] == 0
    assert int((out["cow_dst"] >= 0).sum()) == copies
    assert set(out["cow_tokens"][out["cow_dst"] >= 0].tolist()) <= {5}
    keep = [n for n in range(3) if not appenders[n] or out["cow_dst"][0, n] < 0]
    assert all(out["table"][0, n, 1] == 9 for n in keep)
    assert out["refcount"][9] == 3 - copies and out["refcount"][7] == 3
    for n in range(3):
        c = out["cow_dst"][0, n]
        if c >= 0:
            assert pool[c * PAGE:c * PAGE + 5].tolist() == list(range(200, 205))   # filled only
            assert (pool[c * PAGE + 5:(c + 1) * PAGE] == -1).all()
            assert out["slot_mapping"][0, n, 0] == c * PAGE + 5


def _tokens_of(table, npg, sl, pool, p, n):
    return [int(pool[table[p, n, i // PAGE] * PAGE + i % PAGE]) for i in range(sl[p, n])]


def test_brute_force_rounds_against_token_lists(orc):
    """R rounds of (resample -> append K+1 tokens) on P prompts x N particles vs a plain
    list-of-tokens model; checks every slot written is exclusive to its particle, refcount
    conservation (sum refcounts = sum list lengths) and that resampling moves no
    content (only the append's copy-on-write copies tokens)."""
    rng = np.random.default_rng(0)
    P, N, K, R, MP, NUM = 2, 6, 4, 6, 12, 400
    table, npg, sl, rc = _state(P, N, MP, NUM)
    pool = np.full(NUM * PAGE, -1, np.int32)
    model = [[[] for _ in range(N)] for _ in range(P)]
    # shared prompt of 20 tokens: written once by particle 0, then every particle points at it
    out, (table, npg, sl, rc) = _append(orc, (table, npg, sl, rc), [[20] + [0] * (N - 1)] * P,
                                        pool=pool.view(np.uint8))
    tok = 1
    for p in range(P):
        for j in range(20):
            pool[out["slot_mapping"][p, 0, j]] = tok
            model[p][0].append(tok)
            tok += 1
    a = np.zeros((P, N), np.int32)
    r = orc.kv_reindex_paged(table, npg, rc, a)
    table, npg, rc = r["table"], r["n_pages"], r["refcount"]
    sl = np.take_along_axis(sl, a, 1)
    model = [[list(model[p][0]) for _ in range(N)] for p in range(P)]
    copied = 0
    for rnd in range(R):
        n_new = rng.integers(0, K + 2, size=(P, N)).astype(np.int32)
        before = pool.copy()
        out, (table, npg, sl, rc) = _append(orc, (table, npg, sl, rc), n_new,
                                            pool=pool.view(np.uint8), max_new=K + 1)
        assert out["result"] == 0
        copied += int(out["cow_tokens"].sum())
        slots = out["slot_mapping"][out["slot_mapping"] >= 0]
        assert len(set(slots.tolist())) == slots.size                  # no slot written twice
        assert all(pool[s] == -1 or before[s] == pool[s] for s in slots.tolist())
        for s in slots.tolist():
            assert rc[s // PAGE] == 1                                   # exclusive page
        for p in range(P):
            for n in range(N):
                for j in range(n_new[p, n]):
                    pool[out["slot_mapping"][p, n, j]] = tok
                    model[p][n].append(tok)
                    tok += 1
                assert _tokens_of(table, npg, sl, pool, p, n) == model[p][n]
        assert rc.sum() == sum(int(npg[p, n]) for p in range(P) for n in range(N))
        # resample: the pool's bytes do not change (zero-copy resampling)
        lw = (rng.standard_normal((P, N)) * 1.5).astype(np.float32)
        a = orc.resample(lw, eta=np.inf, seed=rnd)["ancestors"]
        snap = pool.copy()
        r = orc.kv_reindex_paged(table, npg, rc, a)
        assert np.array_equal(pool, snap)
        table, npg, rc = r["table"], r["n_pages"], r["refcount"]
        sl = np.take_along_axis(sl, a, 1)
        model = [[list(model[p][a[p, n]]) for n in range(N)] for p in range(P)]
        for p in range(P):
            for n in range(N):
                assert _tokens_of(table, npg, sl, pool, p, n) == model[p][n]
    assert copied > 0                                                   # copy-on-write exercised


def test_all_or_nothing_failures(orc):
    table, npg, sl, rc = _state(2, 2, 2, 3)
    out, _ = _append(orc, (table, npg, sl, rc), [[PAGE, PAGE], [PAGE, PAGE]])     # 4 pages > 3
    assert out["result"] == 1 and out["status"].tolist() == [128, 128]
    assert (out["refcount"] == 0).all() and (out["n_pages"] == 0).all()
    assert (out["cow_dst"] == -1).all() and (out["cow_src"] == -1).all() and (out["cow_tokens"] == 0).all()
    out, _ = _append(orc, (table, npg, sl, rc), [[0, 3 * PAGE], [0, 0]])          # > max_pages
    assert out["result"] == 1 and out["status"].tolist() == [16, 0]
    npg2 = npg.copy(); npg2[1, 0] = 1                                              # inconsistent
    out, _ = _append(orc, (table, npg2, sl, rc), [[1, 0], [0, 0]])
    assert out["result"] == 1 and out["status"].tolist() == [0, 16]


def test_prefix_sharing_memory_reduction(orc):
    """SPEC.md:486 example: N = 8, K = 16, 16-token pages, 8 rounds each ending in a resample to
    one particle: peak unique pages < half of the no-sharing layout (every particle its own
    copy of its whole sequence)."""
    P, N, K, R, MP, NUM = 1, 8, 16, 8, 40, 2000
    table, npg, sl, rc = _state(P, N, MP, NUM)
    out, (table, npg, sl, rc) = _append(orc, (table, npg, sl, rc), [[64] + [0] * (N - 1)])
    r = orc.kv_reindex_paged(table, npg, rc, np.zeros((1, N), np.int32))
    table, npg, rc = r["table"], r["n_pages"], r["refcount"]
    sl = np.full((1, N), 64, np.int32)
    peak_unique, naive = 0, 0
    for rnd in range(R):
        out, (table, npg, sl, rc) = _append(orc, (table, npg, sl, rc), np.full((1, N), K + 1),
                                            max_new=K + 1)
        assert out["result"] == 0
        peak_unique = max(peak_unique, int((rc > 0).sum()))
        naive = max(naive, int(sum((int(s) + PAGE - 1) // PAGE for s in sl[0])))
        a = np.full((1, N), rnd % N, np.int32)
        r = orc.kv_reindex_paged(table, npg, rc, a)
        table, npg, rc = r["table"], r["n_pages"], r["refcount"]
        sl = np.take_along_axis(sl, a, 1)
    assert peak_unique <= naive and 1 - peak_unique / naive > 0.5
