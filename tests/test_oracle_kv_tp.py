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
