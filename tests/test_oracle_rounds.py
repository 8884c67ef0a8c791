"""Multi-round pin of the oracle (SURVEY.md 8(c) "multi-round trajectories"): R rounds of
Alg. 1 composed from oracle.weights / oracle.resample / oracle.bonus / oracle.kv_reindex on a
toy Markov LM satisfy SMC's unbiasedness identity E[Z_R sum_n wbar_n 1{x_n = s}] = p(s) for
every sequence s, with p(s) exact (tests/smc_rounds.py).  Pinned against the mathematics of
SMC, not against the CUDA path."""
import math

import numpy as np
import pytest

import smc_rounds as sr


def _oracle_backend(orc, P, N, K, seed):
    def backend(r, lp, lq, tok, eta):
        w = orc.weights(lp, lq, tok, V=sr.V, logw_prev=np.full((P, N), orc.neg_log_n(N), np.float32))
        rs = orc.resample(w["logw"], eta=eta, seed=seed, step=r)
        b = orc.bonus(lp, K=K, V=sr.V, seed=seed, step=r, seg=8192)
        assert (w["status"] == 0).all() and (b["status"] == 0).all()
        return w["lse"], b["bonus"], rs["slot_src"], w["logw"]

    def reindex(hist, slot_src):
        h = np.ascontiguousarray(hist)
        T = h.shape[2]
        orc.kv_reindex(h, h, slot_src, n_outer=1, outer_stride=0, prompt_stride=N * T * 4,
                       particle_stride=T * 4, seg_count=1, seg_bytes=T * 4, seg_stride=T * 4)
        return h
    return backend, reindex


@pytest.mark.parametrize("N,K,R", [(8, 1, 2), (4, 2, 2), (1, 1, 2)])
def test_oracle_multi_round_unbiased(orc, N, K, R):
    P = 6000
    p_tab, q_tab = sr.tables()
    backend, reindex = _oracle_backend(orc, P, N, K, seed=0x5EED5EED)
    log_z, hist, wbar = sr.run(backend, reindex, P=P, N=N, K=K, R=R, seed=11, p_tab=p_tab, q_tab=q_tab)
    ev, ps = sr.exact_events(p_tab, R * (K + 1))
    est, se = sr.estimate(log_z, hist, wbar, ev)
    z = (est - ps) / se
    assert np.max(np.abs(z)) < 5.0, (np.max(np.abs(z)), ev[int(np.argmax(np.abs(z)))])
    chi2 = float(np.sum(z ** 2))                  # events are correlated: a loose global bound
    assert chi2 < 3.0 * len(ev), chi2


def test_multi_round_identity_detects_missing_resampling(orc):
    """Negative control: keeping every particle's own history (no S9 reindex) while still
    resetting the weights breaks the identity -- so the pin has power against that bug."""
    P, N, K, R = 6000, 8, 1, 2
    p_tab, q_tab = sr.tables()
    backend, _ = _oracle_backend(orc, P, N, K, seed=0x5EED5EED)
    log_z, hist, wbar = sr.run(backend, lambda h, s: h, P=P, N=N, K=K, R=R, seed=11,
                               p_tab=p_tab, q_tab=q_tab)
    ev, ps = sr.exact_events(p_tab, R * (K + 1))
    est, se = sr.estimate(log_z, hist, wbar, ev)
    z = (est - ps) / se
    assert np.max(np.abs(z)) > 8.0, np.max(np.abs(z))
