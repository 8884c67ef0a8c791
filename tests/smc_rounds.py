"""Multi-round SMC-SD on a toy first-order Markov LM (test harness, no method arithmetic).

Drives R rounds of Alg. 1 through a pluggable backend -- the CPU oracle or
the CUDA library -- and returns what the unbiasedness identity of SMC needs:

    E[ Z_R * sum_n wbar_n 1{x_n = s} ] = p(s)     for every sequence s,     (*)

where Z_R = prod_r (1/N) sum_n w_n^(r) is the SMC estimate of the normalising constant (here 1:
the target is a normalised LM), read from each round's lse = log sum_n exp(lam'_n) with
lam_prev = -ln N after every reset, and wbar the normalised weights of the last round, which
does not resample (eta = 0).  (*) holds for any conditionally unbiased resampling (systematic
and multinomial both are) and fails if the weights, the normalisation, the ancestor draw, the
slot plan / history reindex or the bonus draw is wrong -- e.g. keeping every particle's own
history instead of its ancestor's biases it.  p(s) is exact: a product of table entries.

The draft phase (sampling d ~ q) is out of the path's scope, so the harness
does it with numpy; the bonus token is drawn by the backend (Alg. 1).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

V = 3                     # vocabulary; token V is BOS (first context only)


def tables(seed: int = 7, mismatch: float = 0.8):
    """Target and draft next-token tables [V+1][V] (row = previous token, V = BOS)."""
    rng = np.random.default_rng(seed)
    zp = rng.normal(0.0, 1.0, (V + 1, V))
    zq = zp + mismatch * rng.normal(0.0, 1.0, (V + 1, V))
    p = np.exp(zp) / np.exp(zp).sum(1, keepdims=True)
    q = np.exp(zq) / np.exp(zq).sum(1, keepdims=True)
    return p, q


def exact_target(p_tab, length: int):
    """p(s) for every sequence s in V^length (first-order chain from BOS)."""
    seqs = list(itertools.product(range(V), repeat=length))
    probs = []
    for s in seqs:
        pr, prev = 1.0, V
        for t in s:
            pr *= p_tab[prev, t]
            prev = t
        probs.append(pr)
    return seqs, np.array(probs)


def run(backend, reindex, *, P: int, N: int, K: int, R: int, seed: int, p_tab, q_tab):
    """R rounds for P independent prompts.  backend(r, lp, lq, tok, eta) performs S1-S7 of
    round r on float32 logits lp [P][N][K+1][4], lq [P][N][K][4] (column 3 is padding, NaN)
    and returns (lse [P], bonus [P][N], slot_src [P][N], logw_pre [P][N]); reindex(hist,
    slot_src) applies S9 (in-place slot plan) to the int32 histories [P][N][T] and returns them.
    Returns (log_Z [P], final histories [P][N][R(K+1)], final wbar [P][N])."""
    rng = np.random.default_rng(seed)
    T = R * (K + 1)
    hist = np.zeros((P, N, T), np.int32)
    log_z = np.zeros(P)
    logq_tab, logp_tab = np.log(q_tab), np.log(p_tab)
    wbar = None
    for r in range(R):
        prev = np.full((P, N), V, np.int64) if r == 0 else hist[:, :, r * (K + 1) - 1].astype(np.int64)
        tok = np.zeros((P, N, K), np.int32)
        lp = np.full((P, N, K + 1, 4), np.nan, np.float32)
        lq = np.full((P, N, K, 4), np.nan, np.float32)
        for j in range(K):
            cdf = np.cumsum(q_tab[prev], axis=-1)                   # draft: d_j ~ q(. | prev)
            u = rng.random((P, N, 1))
            d = np.minimum((u > cdf).sum(-1), V - 1)
            tok[:, :, j] = d
            lq[:, :, j, :V] = logq_tab[prev]
            lp[:, :, j, :V] = logp_tab[prev]
            prev = d
        lp[:, :, K, :V] = logp_tab[prev]                            # bonus row p(. | x d)
        last = r == R - 1
        lse, bonus, slot_src, logw_pre = backend(r, lp, lq, tok, 0.0 if last else math.inf)
        log_z += np.asarray(lse, np.float64)
        hist[:, :, r * (K + 1): r * (K + 1) + K] = tok
        hist[:, :, r * (K + 1) + K] = bonus
        if not last:                                                # x^(n) <- x^(a_n) d^(a_n) x+_(a_n)
            hist = reindex(hist, np.asarray(slot_src, np.int32))
        else:
            lw = np.asarray(logw_pre, np.float64)
            m = lw.max(axis=1, keepdims=True)
            e = np.exp(lw - m)
            wbar = e / e.sum(axis=1, keepdims=True)
    return log_z, hist, wbar


def events(length: int):
    """Test functions phi for (*): one-token marginals (position t, token v) and adjacent
    pairs (t, v, v') -- each has a probability large enough for a reliable standard error
    (full sequences would be too rare at V^length outcomes)."""
    ev = [("tok", t, v) for t in range(length) for v in range(V)]
    ev += [("pair", t, v, w) for t in range(length - 1) for v in range(V) for w in range(V)]
    return ev


def phi(ev, seq) -> float:
    if ev[0] == "tok":
        return float(seq[ev[1]] == ev[2])
    return float(seq[ev[1]] == ev[2] and seq[ev[1] + 1] == ev[3])


def exact_events(p_tab, length: int):
    """E_p[phi] for every event, by enumerating V^length sequences."""
    seqs, ps = exact_target(p_tab, length)
    ev = events(length)
    return ev, np.array([sum(pr * phi(e, s) for s, pr in zip(seqs, ps)) for e in ev])


def estimate(log_z, hist, wbar, ev):
    """Per-event mean and standard error of Z * sum_n wbar_n phi(x_n) over the prompts."""
    P, N, T = hist.shape
    z = np.exp(log_z)
    contrib = np.zeros((P, len(ev)))
    for k, e in enumerate(ev):
        if e[0] == "tok":
            ind = (hist[:, :, e[1]] == e[2]).astype(np.float64)
        else:
            ind = ((hist[:, :, e[1]] == e[2]) & (hist[:, :, e[1] + 1] == e[3])).astype(np.float64)
        contrib[:, k] = z * (wbar * ind).sum(axis=1)
    return contrib.mean(0), contrib.std(0, ddof=1) / math.sqrt(P)
