"""Pins for the oracle's S3 (reweight) and S4 (normalise + ESS) via smcsd_weights.

Pins: special cases with closed forms, brute-force enumeration
of tiny V^K block spaces (tower property E_q[w] = 1; i.i.d. product
form), worked ESS values and the
ESS-rate theorem at N = 10^4.
"""
import itertools
import math

import numpy as np
import pytest

import synth
from conftest import read_golden


def _rows(probs, ld=None):
    """fp32 logit rows z = ln(prob) (padded to ld with NaN that must never be read)."""
    probs = np.asarray(probs, dtype=np.float64)
    V = probs.shape[-1]
    ld = ld or (V + 3) // 4 * 4
    with np.errstate(divide="ignore"):
        z = np.log(probs).astype(np.float32)
    out = np.full(probs.shape[:-1] + (ld,), np.nan, dtype=np.float32)
    out[..., :V] = z
    return out


def test_identical_models_give_zero_increment(orc):
    # q == p  =>  every ratio is 1, Delta = 0 exactly, ESS = N
    lp, lq, tok = synth.lm_logits(2, 8, 4, 1000, dtype=synth.torch.float32, sigma_d=0.0, seed=11)
    lq_same = lp[:, :, :4, :].contiguous()
    prev = synth.random_logw(2, 8, seed=5).numpy()
    out = orc.weights(lp.numpy(), lq_same.numpy(), tok.numpy(), V=1000, logw_prev=prev)
    assert np.array_equal(out["logw"], prev)
    both = out["logp_tok"] - out["logq_tok"]
    assert np.all(both == 0.0)
    prev_u = np.full((2, 8), np.float32(-math.log(8)))
    out = orc.weights(lp.numpy(), lq_same.numpy(), tok.numpy(), V=1000, logw_prev=prev_u)
    assert np.all(out["ess"] == 8.0)


def test_single_particle_single_token(orc):
    # K=1, N=1: weight = log p(d)/q(d)
    p = [0.1, 0.6, 0.3]
    q = [0.3, 0.3, 0.4]
    lp = _rows([[[p, [1 / 3] * 3]]])        # [P=1][N=1][K+1=2][ld]
    lq = _rows([[[q]]])
    tok = np.array([[[1]]], dtype=np.int32)
    out = orc.weights(lp, lq, tok, V=3, logw_prev=np.zeros((1, 1), np.float32))
    assert out["logw"][0, 0] == pytest.approx(math.log(0.6 / 0.3), abs=1e-6)
    assert out["ess"][0] == 1.0
    assert out["lse"][0] == pytest.approx(math.log(2.0), abs=1e-6)


def test_power_weight_examples(orc):
    # alpha*log p - log q
    lp = _rows([[[[0.5, 0.5]]]])
    lq = _rows([[[[0.25, 0.75]]]])
    tok = np.array([[[0]]], dtype=np.int32)
    z = np.zeros((1, 1), np.float32)
    out = orc.weights(lp, lq, tok, V=2, logw_prev=z, alpha=2.0)
    assert out["logw"][0, 0] == pytest.approx(0.0, abs=1e-7)      # 0.5^2 / 0.25 = 1
    out1 = orc.weights(lp, lq, tok, V=2, logw_prev=z, alpha=1.0)
    assert out1["logw"][0, 0] == pytest.approx(math.log(2.0), abs=1e-7)
    # p = q, any alpha: (alpha - 1) log p
    for alpha in (0.5, 1.0, 3.0):
        o = orc.weights(lp, lp, tok, V=2, logw_prev=z, alpha=alpha)
        assert o["logw"][0, 0] == pytest.approx((alpha - 1) * math.log(0.5), abs=1e-6)


def _enumeration_fixture(V, K, seed, prefix_dependent=True):
    """Tabular draft/target LMs over V tokens, one row per prefix (or per position)."""
    n_pref = sum(V ** j for j in range(K)) if prefix_dependent else K
    tp = synth.dirichlet_rows(n_pref, V, seed=seed).numpy()
    tq = synth.dirichlet_rows(n_pref, V, seed=seed + 1, conc=2.0).numpy()

    def row_index(prefix):
        if not prefix_dependent:
            return len(prefix)
        off = sum(V ** j for j in range(len(prefix)))
        idx = 0
        for t in prefix:
            idx = idx * V + t
        return off + idx

    blocks = list(itertools.product(range(V), repeat=K))
    N = len(blocks)
    P_rows = np.zeros((1, N, K + 1, V))
    Q_rows = np.zeros((1, N, K, V))
    tok = np.zeros((1, N, K), np.int32)
    logq_block = np.zeros(N)
    logp_block = np.zeros(N)
    for n, d in enumerate(blocks):
        for j in range(K):
            r = row_index(d[:j])
            P_rows[0, n, j] = tp[r]
            Q_rows[0, n, j] = tq[r]
            tok[0, n, j] = d[j]
            logq_block[n] += math.log(tq[r][d[j]])
            logp_block[n] += math.log(tp[r][d[j]])
        P_rows[0, n, K] = 1.0 / V                       # bonus row: never read
    return _rows(P_rows), _rows(Q_rows), tok, logp_block, logq_block


@pytest.mark.parametrize("V,K", [(4, 3), (3, 4), (2, 6)])
def test_enumeration_tower_property(orc, V, K):
    # lam_prev = ln q(d) => lam' = ln p(d) and lse = ln sum_d p(d) = 0 (E_q[w] = 1,
    # PAPER.md:928, 1450).  One particle per block d in V^K.
    lp, lq, tok, logp_block, logq_block = _enumeration_fixture(V, K, seed=100 + V)
    prev = logq_block.astype(np.float32)[None, :]
    out = orc.weights(lp, lq, tok, V=V, logw_prev=prev)
    assert out["status"][0] == 0
    assert out["lse"][0] == pytest.approx(0.0, abs=1e-6)
    assert np.allclose(out["logw"][0], logp_block, atol=2e-6)


@pytest.mark.parametrize("V,K", [(4, 3), (3, 4)])
def test_enumeration_iid_second_moment(orc, V, K):
    # one fixed row per position: sum_d q(d) w(d)^2 = prod_j sum_v p_j^2 / q_j
    # (PAPER.md:1194-1207), and sum_d q(d) w(d) = 1
    lp, lq, tok, logp_block, logq_block = _enumeration_fixture(V, K, seed=7, prefix_dependent=False)
    N = tok.shape[1]
    out = orc.weights(lp, lq, tok, V=V, logw_prev=np.zeros((1, N), np.float32))
    w = np.exp(out["logw"][0].astype(np.float64))
    qd = np.exp(logq_block)
    tp = np.exp(lp[0, 0, :K, :V].astype(np.float64))
    tq = np.exp(lq[0, 0, :K, :V].astype(np.float64))
    tp /= tp.sum(1, keepdims=True)
    tq /= tq.sum(1, keepdims=True)
    prod = np.prod((tp ** 2 / tq).sum(1))
    assert np.sum(qd * w) == pytest.approx(1.0, rel=1e-6)
    assert np.sum(qd * w * w) == pytest.approx(prod, rel=1e-6)


def test_ess_worked_values(orc):
    for line in read_golden("ess_worked.txt"):
        lhs, rest = line.split("->")
        want = float(rest.split(";")[0])
        w = np.array([float(x) for x in lhs.split(",")])
        N = len(w)
        with np.errstate(divide="ignore"):
            lw = np.log(w).astype(np.float32)[None, :]
        out = orc.resample(lw, eta=0.0)         # eta = 0: never resample, just S4
        assert out["ess"][0] == pytest.approx(want, rel=1e-7), line
        assert out["resampled"][0] == 0


def test_ess_bounds_random(orc):
    rng = np.random.default_rng(9)
    for N in (1, 2, 7, 64, 1000):
        lw = (rng.standard_normal((3, N)) * 3).astype(np.float32)
        out = orc.resample(lw, eta=0.0)
        assert np.all(out["ess"] >= 1.0 - 1e-12) and np.all(out["ess"] <= N + 1e-9)
        assert np.allclose(out["wnorm"].sum(1), 1.0, atol=1e-12)


def _iid_rate_fixture(K, N, seed):
    lp_row = _rows([0.5, 0.5])
    lq_row = _rows([0.25, 0.75])
    rng = np.random.default_rng(seed)
    tok = (rng.random((1, N, K)) < 0.75).astype(np.int32)     # d ~ q = (0.25, 0.75)
    lp = np.broadcast_to(lp_row, (1, N, K + 1, lp_row.shape[-1])).copy()
    lq = np.broadcast_to(lq_row, (1, N, K, lq_row.shape[-1])).copy()
    return lp, lq, tok


def test_ess_rate_theorem(orc):
    # ESS/N -> 1/(1+chi2(p_K||q_K)) = (1 + 1/3)^-K for the i.i.d. pair (
    # SPEC.md:203, 323): K=2 -> 0.5625
    N = 10000
    lp, lq, tok = _iid_rate_fixture(2, N, seed=31)
    out = orc.weights(lp, lq, tok, V=2, logw_prev=np.zeros((1, N), np.float32))
    assert out["ess"][0] / N == pytest.approx(0.5625, abs=0.02)
    # bonus-gain corollary: K vs K+1 drafted tokens
    lp3, lq3, tok3 = _iid_rate_fixture(3, N, seed=32)
    out3 = orc.weights(lp3, lq3, tok3, V=2, logw_prev=np.zeros((1, N), np.float32))
    ratio = (out["ess"][0] / N) / (out3["ess"][0] / N)
    assert ratio == pytest.approx(4.0 / 3.0, rel=0.05)


def test_n_drafted_rows_beyond_are_not_read(orc):
    # EOS inside a block (reading G10): rows j >= k_n are never read -- fill them with NaN
    lp, lq, tok = synth.lm_logits(1, 4, 4, 100, dtype=synth.torch.float32, seed=3)
    lp, lq, tok = lp.numpy(), lq.numpy(), tok.numpy()
    nd = np.array([[4, 2, 0, 3]], np.int32)
    ref = orc.weights(lp, lq, tok, V=100, n_drafted=nd)
    for n in range(4):
        lp[0, n, nd[0, n]:, :] = np.nan
        lq[0, n, nd[0, n]:, :] = np.nan
        tok[0, n, nd[0, n]:] = -7
    out = orc.weights(lp, lq, tok, V=100, n_drafted=nd)
    assert out["status"][0] == 0
    assert np.array_equal(out["logw"], ref["logw"])
    assert out["logw"][0, 2] == np.float32(-math.log(4))            # k_n = 0: weight kept


def test_status_flags(orc):
    lp, lq, tok = synth.lm_logits(1, 4, 2, 64, dtype=synth.torch.float32, seed=4)
    lp, lq, tok = lp.numpy(), lq.numpy(), tok.numpy()
    base = orc.weights(lp, lq, tok, V=64)
    assert base["status"][0] == 0
    t2 = tok.copy(); t2[0, 1, 0] = 64
    o = orc.weights(lp, lq, t2, V=64)
    assert o["status"][0] == orc.ST_BAD_TOKEN and o["logw"][0, 1] == -np.inf
    q2 = lq.copy(); q2[0, 2, 1, tok[0, 2, 1]] = -np.inf
    o = orc.weights(lp, q2, tok, V=64)
    assert o["status"][0] == orc.ST_NOT_ABSCONT and o["logw"][0, 2] == -np.inf
    p2 = lp.copy(); p2[0, 3, 0, 5] = np.nan
    o = orc.weights(p2, lq, tok, V=64)
    assert o["status"][0] == orc.ST_NONFINITE and o["logw"][0, 3] == -np.inf
    p3 = lp.copy(); p3[0, 0, 0, tok[0, 0, 0]] = -np.inf     # p(d) = 0: weight 0, no flag
    o = orc.weights(p3, lq, tok, V=64)
    assert o["status"][0] == 0 and o["logw"][0, 0] == -np.inf
    allbad = np.full((1, 4), -np.inf, np.float32)
    o = orc.weights(lp, lq, tok, V=64, logw_prev=allbad)
    assert o["status"][0] == orc.ST_DEGENERATE and o["lse"][0] == -np.inf and o["ess"][0] == 0.0


# ------------------------------------------------------------- PowerSMC (NEXT #4, App. F)
def test_powersmc_closed_forms(orc):
    # alpha = 1: per-token weight = log sum p = 0
    rng = np.random.default_rng(3)
    lg = (rng.standard_normal((2, 5, 1, 1000)) * 3).astype(np.float32)
    out = orc.powersmc_weights(lg, alpha=1.0, logw_prev=np.zeros((2, 5), np.float32))
    assert np.allclose(out["inc"], 0.0, atol=1e-12)
    # alpha = 2, single-position p = (0.6, 0.4): sum p^2 = 0.52
    row = np.log(np.array([[[[0.6, 0.4, np.nan, np.nan]]]])).astype(np.float32)
    out = orc.powersmc_weights(row, V=2, alpha=2.0, logw_prev=np.zeros((1, 1), np.float32))
    assert out["inc"][0, 0] == pytest.approx(math.log(0.6 ** 2 + 0.4 ** 2), abs=1e-7)
    # uniform row: sum (1/V)^alpha = V^(1 - alpha)
    for V, a in ((1000, 0.5), (128, 3.0)):
        u = np.zeros((1, 1, 1, V), np.float32)
        out = orc.powersmc_weights(u, alpha=a, logw_prev=np.zeros((1, 1), np.float32))
        assert out["inc"][0, 0] == pytest.approx((1 - a) * math.log(V), abs=1e-10)


def test_powersmc_matches_scipy(orc):
    from scipy.special import logsumexp, log_softmax
    rng = np.random.default_rng(8)
    lg = (rng.standard_normal((1, 3, 2, 3000)) * 2.5).astype(np.float32)
    for a, tau in ((0.5, 1.0), (4.0, 0.7)):
        out = orc.powersmc_weights(lg, alpha=a, tau=tau, logw_prev=np.zeros((1, 3), np.float32))
        for n in range(3):
            lp = log_softmax(tau * lg[0, n, 0].astype(np.float64))
            assert out["inc"][0, n] == pytest.approx(logsumexp(a * lp), abs=1e-10)


def test_openmp_timing_build_is_bit_identical(orc):
    """liboracle_omp.so (the timing-only -fopenmp build used by bench.py's cpu_baseline) gives
    the same bits as the plain build: the rows of S1+S2 are independent and S3/S4 stay serial."""
    import torch
    import synth
    lp, lq, tok = synth.lm_logits(3, 9, 5, 20001, dtype=torch.bfloat16, seed=12)
    u16 = lambda t: t.view(torch.int16).numpy().view(np.uint16)
    nd = np.array([[5, 0, 3, 5, 5, 9, 5, 1, 5]] * 3, np.int32)
    a = orc.weights(u16(lp), u16(lq), tok.numpy(), n_drafted=nd, alpha=1.5)
    try:
        assert orc.set_threads(4) >= 1
        b = orc.weights(u16(lp), u16(lq), tok.numpy(), n_drafted=nd, alpha=1.5)
    finally:
        orc.set_threads(1)
    for k in a:
        assert np.array_equal(a[k], b[k], equal_nan=True), k
