"""Pins for the oracle's S8/S9 byte reindex and the TP (vocab-shard) partial/combine.

S8/S9 are checked against numpy fancy indexing (an independent gather); the TP merge is
checked against the unsharded row log-softmax (exact up to fp64 rounding).
"""
import math

import numpy as np
import pytest

import synth


def _kv(L, P, N, H, S, d, seed):
    return synth.kv_bits((L, 2, P, N, H, S, d), seed=seed).numpy()


def _geom(kv, S_fill=None):
    L, C, P, N, H, S, d = kv.shape
    e = kv.itemsize
    S_fill = S if S_fill is None else S_fill
    return dict(n_outer=L * C, outer_stride=P * N * H * S * d * e, prompt_stride=N * H * S * d * e,
                particle_stride=H * S * d * e, seg_count=H, seg_bytes=S_fill * d * e,
                seg_stride=S * d * e)


def test_kv_out_of_place_matches_fancy_index(orc):
    src = _kv(2, 2, 4, 2, 64, 16, seed=1)                     # cfg1 toy KV: 2 layers, seq 64
    a = np.array([[0, 0, 3, 3], [1, 2, 2, 2]], np.int32)
    dst = np.zeros_like(src)
    orc.kv_reindex(dst, src, a, **_geom(src))
    want = np.stack([src[:, :, p][:, :, a[p]] for p in range(2)], axis=2)
    assert np.array_equal(dst, want)


def test_kv_identity_and_partial_fill(orc):
    src = _kv(2, 1, 4, 2, 64, 16, seed=2)
    dst = np.zeros_like(src)
    orc.kv_reindex(dst, src, np.arange(4, dtype=np.int32)[None], **_geom(src))
    assert np.array_equal(dst, src)
    # only the filled prefix [0, 40) of each head is copied (reading G12)
    dst = np.zeros_like(src)
    a = np.array([[3, 3, 1, 0]], np.int32)
    orc.kv_reindex(dst, src, a, **_geom(src, S_fill=40))
    assert np.array_equal(dst[..., :40, :], src[:, :, :, a[0]][..., :40, :])
    assert np.all(dst[..., 40:, :] == 0)


def test_kv_in_place_slot_plan(orc):
    rng = np.random.default_rng(3)
    for _ in range(20):
        N = 8
        lw = (rng.standard_normal((1, N)) * 2).astype(np.float32)
        r = orc.resample(lw, eta=np.inf, seed=int(rng.integers(1 << 40)))
        kv = _kv(2, 1, N, 2, 8, 16, seed=int(rng.integers(1 << 20)))
        before = kv.copy()
        orc.kv_reindex(kv, kv, r["slot_src"], **_geom(kv))
        s = r["slot_src"][0]
        assert np.array_equal(kv, before[:, :, :, s])
        # the out-of-place result with the sorted ancestors is the same multiset of blocks
        out = np.zeros_like(before)
        orc.kv_reindex(out, before, r["ancestors"], **_geom(before))
        key = lambda x: sorted(x[:, :, 0, n].tobytes() for n in range(N))
        assert key(out) == key(kv)


def test_kv_invalid_index_policy(orc):
    """Reading G23: an out-of-range entry is skipped (its destination untouched) and flags
    ST_BAD_INDEX; an in-place plan whose source is itself a destination is not hazard-free
    (SPEC.md:466-474 copies are defined only for a valid ancestor vector) -- the prompt is
    flagged and left untouched.  Valid prompts of the same call are unaffected."""
    src = _kv(1, 3, 4, 1, 4, 16, seed=5)
    dst = np.zeros_like(src)
    a = np.array([[1, 4, 2, -1], [0, 0, 1, 1], [3, 3, 3, 3]], np.int32)
    st = orc.kv_reindex(dst, src, a, **_geom(src))
    assert st.tolist() == [orc.ST_BAD_INDEX, 0, 0]
    assert np.array_equal(dst[:, :, 0, 0], src[:, :, 0, 1]) and np.array_equal(dst[:, :, 0, 2], src[:, :, 0, 2])
    assert np.all(dst[:, :, 0, 1] == 0) and np.all(dst[:, :, 0, 3] == 0)       # skipped entries
    assert np.array_equal(dst[:, :, 1], src[:, :, 1][:, :, [0, 0, 1, 1]])
    # out-of-place, [0,0,1,1] is a fine ancestor vector; in place it overwrites source 1
    kv = _kv(1, 2, 4, 1, 4, 16, seed=6)
    before = kv.copy()
    st = orc.kv_reindex(kv, kv, np.array([[0, 0, 1, 1], [0, 0, 2, 3]], np.int32), **_geom(kv))
    assert st.tolist() == [orc.ST_BAD_INDEX, 0]
    assert np.array_equal(kv[:, :, 0], before[:, :, 0])                          # untouched
    assert np.array_equal(kv[:, :, 1], before[:, :, 1][:, :, [0, 0, 2, 3]])


def test_tp_partials_merge_to_unsharded(orc):
    rng = np.random.default_rng(4)
    V = 1000
    for dtype in (np.float32, np.uint16):
        row = (rng.standard_normal(V) * 3).astype(np.float32)
        if dtype == np.uint16:
            row = (row.view(np.uint32) >> 16).astype(np.uint16)
        row[17] = row[17]  # noqa
        for G in (1, 2, 3, 8):
            bounds = np.linspace(0, V, G + 1).astype(int)
            for d in (0, 499, 999):
                parts = np.stack([orc.row_partial(row[bounds[g]:bounds[g + 1]], bounds[g], d, tau=0.7)[0]
                                  for g in range(G)])
                ell, flag = orc.combine_partials(parts)
                ref, _ = orc.row_logprob(row, d, tau=0.7)
                assert flag == 0
                assert ell == pytest.approx(ref, abs=1e-12)


def test_tp_masked_shard(orc):
    row = np.array([1.0, 2.0, -np.inf, -np.inf], np.float32)
    p0, _ = orc.row_partial(row[:2], 0, 1)
    p1, _ = orc.row_partial(row[2:], 2, 1)
    assert p1[0] == -np.inf and p1[1] == 0.0 and p1[2] == -np.inf
    ell, flag = orc.combine_partials(np.stack([p0, p1]))
    assert flag == 0 and ell == pytest.approx(2.0 - math.log(math.e + math.e ** 2), abs=1e-14)


# ------------------------------------------------------------- paged reindex (NEXT #1)
def _paged_fixture(P, N, pages_per, seed, shared_prefix=2):
    """Particles of a prompt share `shared_prefix` prompt pages, then own their pages."""
    rng = np.random.default_rng(seed)
    MP = pages_per + 2
    table = np.full((P, N, MP), -1, np.int32)
    n_pages = np.zeros((P, N), np.int32)
    nxt = 0
    refc = []
    for p in range(P):
        prefix = list(range(nxt, nxt + shared_prefix)); nxt += shared_prefix
        refc += [N] * shared_prefix
        for n in range(N):
            own = int(rng.integers(0, pages_per + 1))
            ids = prefix + list(range(nxt, nxt + own)); nxt += own
            refc += [1] * own
            table[p, n, :len(ids)] = ids
            n_pages[p, n] = len(ids)
    return table, n_pages, np.array(refc, np.int32)


def test_paged_identity_and_resample_to_one(orc):
    table, n_pages, rc = _paged_fixture(1, 6, 4, seed=1)
    out = orc.kv_reindex_paged(table, n_pages, rc, np.arange(6, dtype=np.int32)[None])
    assert np.array_equal(out["refcount"], rc) and not out["freed"].any()
    assert np.array_equal(out["table"], table)
    # all ancestors = particle 1: its pages reach refcount N, others' freed
    a = np.full((1, 6), 1, np.int32)
    out = orc.kv_reindex_paged(table, n_pages, rc, a)
    own1 = [pg for pg in table[0, 1, :n_pages[0, 1]] if rc[pg] == 1]
    assert all(out["refcount"][pg] == 6 for pg in own1)
    others = [pg for n in range(6) if n != 1 for pg in table[0, n, :n_pages[0, n]] if rc[pg] == 1]
    assert all(out["freed"][pg] == 1 and out["refcount"][pg] == 0 for pg in others)
    assert all(out["refcount"][pg] == 6 for pg in table[0, 0, :2])           # shared prefix
    assert np.all(out["table"][0] == table[0, 1])


def test_paged_conservation_random(orc):
    rng = np.random.default_rng(5)
    for trial in range(40):
        P, N = int(rng.integers(1, 4)), int(rng.integers(1, 40))
        table, n_pages, rc = _paged_fixture(P, N, 8, seed=trial)
        lw = (rng.standard_normal((P, N)) * 2).astype(np.float32)
        a = orc.resample(lw, eta=np.inf, seed=trial)["ancestors"]
        out = orc.kv_reindex_paged(table, n_pages, rc, a)
        # refcount conservation: total references = total list lengths
        assert out["refcount"].sum() == out["n_pages"].sum()
        assert rc.sum() == n_pages.sum()
        # the new lists are the ancestors' lists (independent gather)
        for p in range(P):
            assert np.array_equal(out["n_pages"][p], n_pages[p][a[p]])
            for n in range(N):
                L = n_pages[p, a[p, n]]
                assert np.array_equal(out["table"][p, n, :L], table[p, a[p, n], :L])
        # every page's refcount = its number of occurrences in the new tables
        cnt = np.bincount(out["table"][out["table"] >= 0].ravel(), minlength=rc.size)
        assert np.array_equal(cnt, out["refcount"])
        assert np.array_equal(out["freed"] == 1, (rc > 0) & (out["refcount"] == 0))
        assert np.all(out["status"] == 0)


def test_paged_bad_ids_flagged(orc):
    table, n_pages, rc = _paged_fixture(1, 4, 3, seed=2)
    t2 = table.copy(); t2[0, 2, 0] = 10 ** 6
    out = orc.kv_reindex_paged(t2, n_pages, rc, np.arange(4, dtype=np.int32)[None])
    assert out["status"][0] == orc.ST_BAD_PAGE
    out = orc.kv_reindex_paged(table, n_pages, rc, np.array([[0, 9, 1, 2]], np.int32))
    assert out["status"][0] == orc.ST_BAD_PAGE
